# GPU parity suite + rows-engine timing / oracle check at full batches
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python tools/rows_check.py --sizes ${S:-36,40,48,56,64,68,72,80,88,96,100,104,112,120,124,128} > gpurun_out/rows_check.jsonl 2>&1
