# GPU parity suite + lyap / sylv sweep lines (device-timed, no CPU / e2e legs)
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
for w in lyap-sweep sylv-sweep; do
  timeout 600 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/sweep_$w.log 2>&1; echo "$w rc=$?"
done
