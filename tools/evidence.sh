#!/bin/bash
# Round-end evidence on one B200: full bench line, ncu launch lists of the
# three sweeps (time + DRAM bytes per launch), ncu --set full of the top
# kernels.  Each ncu command runs only after the same command exited 0.
set -u
O=gpurun_out
python bench.py --steps 10 --warmup 3 --json-out $O/bench_detail.json > $O/bench_final.log 2>&1; echo "bench rc=$?"
for w in chol-sweep lyap-sweep sylv-sweep; do
  CMD="python bench.py --workload $w --steps 1 --warmup 1 --no-cpu --no-e2e --no-extra"
  $CMD > $O/plain_$w.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 300 --csv \
      --log-file $O/launches_$w.csv $CMD > $O/ncu_launch_$w.log 2>&1; echo "launches $w rc=$?"
done
run1() {  # name, run_one args
  local name=$1; shift
  python tools/run_one.py "$@" --reps 2 > $O/plain_$name.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"$KRE" -s 1 -c 1 -o $O/full_$name \
      python tools/run_one.py "$@" --reps 2 > $O/ncu_full_$name.log 2>&1; echo "full $name rc=$?"
}
KRE=chol_rows_kernel run1 chol128 --eq cholesky --n 128 --variant 1 --b 8 --engine rows
KRE=chol_rows_kernel run1 chol92 --eq cholesky --n 92 --variant 1 --b 4 --engine rowsmix
KRE=pipe_kernel run1 sylv128 --eq sylvester --n 128 --variant 13 --b 8 --engine pipe
KRE=pipe_kernel run1 lyap64 --eq lyapunov --n 64 --variant 5 --b 8 --engine pipe
KRE=pipe_kernel run1 sylv64 --eq sylvester --n 64 --variant 13 --b 8 --engine pipe
KRE=pipe_kernel run1 lyap128 --eq lyapunov --n 128 --variant 5 --b 8 --engine pipe
