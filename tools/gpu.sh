#!/bin/bash
# gpurun helper: tools/gpu.sh <timeout_s> '<command>'  (creates gpurun_out/r02 on the box first)
t=$1; shift
exec timeout $((t + 900)) /usr/local/graft/bin/gpurun --timeout "$t" -- "mkdir -p gpurun_out/r02; $*"
