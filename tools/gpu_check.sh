set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
for n in 16 32 64 128; do for m in 0 1 2 3 4 7; do echo "n=$n mode=$m $(LAGEN_WAVE_MODE=$m timeout 120 python tools/run_one.py --eq sylvester --n $n --variant 13 --b 8 --engine wave --reps 2 2>&1 | tail -1)"; done; done > gpurun_out/wave_modes.txt 2>&1
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench exit $?" >> gpurun_out/bench.log
