set -u
O=gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/gpuinfo.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/smoke.log
timeout 900 python bench.py --steps 10 --warmup 3 > $O/bench_final.log 2>&1; echo "bench rc=$?" >> $O/bench_final.log
CMD="python bench.py --workload chol-sweep --steps 1 --warmup 1 --no-cpu --no-e2e --no-extra"
timeout 300 $CMD > $O/plain_chol.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 300 --csv \
      --log-file $O/launches_chol-sweep.csv $CMD > $O/ncu_launch_chol.log 2>&1; echo "launches rc=$?" >> $O/plain_chol.log
