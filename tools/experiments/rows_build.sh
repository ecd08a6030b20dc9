#!/bin/bash
# tools/experiments/rows_build.sh "N B WG F4 tag [extra flags]" ... -> tools/experiments/rows_bin/c_N_tag
mkdir -p tools/experiments/rows_bin
for cfg in "$@"; do
  set -- $cfg
  n=$1; b=$2; wg=$3; f4=$4; tag=$5; shift 5
  out=tools/experiments/rows_bin/c_${n}_${tag}
  nvcc -cudart shared -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++20 --expt-relaxed-constexpr -Xptxas -v -DPN=$n -DPB=$b -DPWG=$wg -DPF4=$f4 "$@" \
     -Iinclude -Ipaper_1906_08613_b200/csrc tools/experiments/rows_bench.cu -o $out 2>&1 | grep -E "error|registers|spill" | grep -v "_Z3gen" | grep -v "^ptxas info    : Function" | grep -v "32 registers\|0 bytes stack" | sed "s/^/$n $tag: /" &
done
wait
