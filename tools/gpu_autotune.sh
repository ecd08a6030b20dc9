# full GPU autotune of the dispatch table (every engine x variant x b per (eq, n))
timeout 2400 python tools/autotune.py --reps 5 > gpurun_out/autotune.log 2>&1; echo "autotune rc=$?" >> gpurun_out/autotune.log
