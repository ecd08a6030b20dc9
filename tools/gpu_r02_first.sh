#!/bin/bash
# round-2 first evidence: parity suite, smoke, bench (+detail), launch lists, ncu full of top kernels
set -u
O=gpurun_out
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/gpuinfo.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" | tee -a $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?" | tee -a $O/smoke.log
bash tools/evidence.sh
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_reference.log 2>&1; echo "ref rc=$?"
tail -c 3000 $O/bench_final.log
