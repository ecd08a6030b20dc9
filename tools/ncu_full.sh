#!/bin/bash
# ncu --set full of one kernel of one batched solve (tools/run_one.py), only
# after the same command exited 0 without ncu.
#   tools/ncu_full.sh <name> <kernel-regex> <run_one args...>
set -u
O=gpurun_out/r02
mkdir -p $O
name=$1; KRE=$2; shift 2
python tools/run_one.py "$@" --reps 2 > $O/plain_$name.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"$KRE" -s 1 -c 1 -o $O/full_$name \
    python tools/run_one.py "$@" --reps 2 > $O/ncu_full_$name.log 2>&1
echo "full $name rc=$?"
