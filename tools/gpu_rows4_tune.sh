# rows-engine b = 4 kernels (unpadded, n = 4 mod 8): WG x work-split sweep
S=36,44,52,60,68,76,84,92,100,108,116,124
for wg in 1 2 4; do for m in 1 5 9 13; do
  LAGEN_ROWS_WG=$wg LAGEN_ROWS_MODE=$m timeout 300 python tools/engine_compare.py --eq cholesky --sizes $S --runs 1:4:rows --reps 3 | sed "s/^/$wg $m /"
done; done > gpurun_out/rows4_tune.txt 2>&1
