# mixed-block rows engine (n = 4 mod 8: partition 4, 8, 8, ...) against the
# padded and the native b = 4 instances: parity first, then a WG x work-split sweep
S=12,20,28,36,44,52,60,68,76,84,92,100,108,116,124
timeout 600 python tools/engine_compare.py --eq cholesky --sizes $S --runs 1:4:generic,1:4:rowsmix,1:4:rowspad,1:4:rows --reps 5 > gpurun_out/rowsmix_ab.txt 2>&1
for wg in 1 2 4; do for m in 1 5 9 13; do
  LAGEN_ROWS_WG=$wg LAGEN_ROWS_MODE=$m timeout 300 python tools/engine_compare.py --eq cholesky --sizes $S --runs 1:4:rowsmix --reps 3 | sed "s/^/$wg $m /"
done; done > gpurun_out/rowsmix_tune.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "cholesky or fixtures or engine" > gpurun_out/rowsmix_pytest.txt 2>&1
tail -3 gpurun_out/rowsmix_pytest.txt
