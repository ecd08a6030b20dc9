#!/bin/bash
# tools/gang_build.sh "N NR P Q MINB" ...  -> tools/experiments/gang_bin/g_N_NR_P_Q_MINB
mkdir -p tools/experiments/gang_bin
for cfg in "$@"; do
  set -- $cfg
  out=tools/experiments/gang_bin/g_$1_$2_$3_$4_$5
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++20 -Xptxas -v -DGN=$1 -DGNR=$2 -DGP=$3 -DGQ=$4 -DGMINB=$5 \
     $GANG_EXTRA -Itools/experiments tools/experiments/gang_bench.cu -o $out 2>&1 | grep -E "error|registers|spill" | grep -v "_Z3gen" | grep -v "^ptxas info    : Function" | sed "s/^/$cfg: /" &
done
wait
