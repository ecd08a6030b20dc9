# rows-engine WG x work-split sweep (b = 8 kernels, n % 8 == 0)
S=40,48,56,64,72,80,88,96,104,112,120,128
for wg in 1 2 4; do for m in 1 5 9 13; do
  LAGEN_ROWS_WG=$wg LAGEN_ROWS_MODE=$m timeout 300 python tools/engine_compare.py --eq cholesky --sizes $S --runs 1:8:rows --reps 3 | sed "s/^/$wg $m /"
done; done > gpurun_out/rows_tune.txt 2>&1
