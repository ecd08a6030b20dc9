# parity + wave-engine timing sweep (one GPU)
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
S=16,24,32,40,48,56,64,72,80,88,96,104,112,120,128
timeout 600 python tools/engine_compare.py --eq sylvester --sizes $S --runs 13:8:wave,13:4:wave > gpurun_out/wave_sylv.jsonl 2>&1
timeout 600 python tools/engine_compare.py --eq lyapunov --sizes $S --runs 5:8:wave,5:4:wave > gpurun_out/wave_lyap.jsonl 2>&1
for n in 32 128; do for m in 0 1 2; do echo "n=$n mode=$m $(LAGEN_WAVE_MODE=$m timeout 120 python tools/run_one.py --eq sylvester --n $n --variant 13 --b 8 --engine wave --reps 2 2>&1 | tail -1)"; done; done > gpurun_out/wave_modes.txt 2>&1
