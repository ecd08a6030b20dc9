# ncu --set full (source-level) of the Cholesky kernels at n = 128 / 64 (rows) and 32 (column)
for n in 128 64 32; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:chol -c 1 -s 2 -o gpurun_out/chol_$n -f \
    python tools/run_one.py --eq cholesky --n $n --reps 2 > gpurun_out/ncu_chol_$n.log 2>&1
done
