#!/bin/bash
# tools/experiments/rsw_build.sh "EQ N tag [extra flags]" ... -> tools/experiments/rsw_bin/r_EQ_N_tag
mkdir -p tools/experiments/rsw_bin
for cfg in "$@"; do
  set -- $cfg
  eq=$1; n=$2; tag=${3:-base}; if [ $# -ge 3 ]; then shift 3; else shift 2; fi
  out=tools/experiments/rsw_bin/r_${eq}_${n}_${tag}
  nvcc -cudart shared -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++20 --expt-relaxed-constexpr -Xptxas -v -DPEQ=$eq -DPN=$n "$@" \
     -Iinclude -Ipaper_1906_08613_b200/csrc tools/experiments/rsw_bench.cu -o $out 2>&1 | grep -E "error|registers|spill" | grep -v "_Z3gen" | grep -v "^ptxas info    : Function" | grep -v "32 registers\|0 bytes stack" | sed "s/^/$eq $n $tag: /" &
done
wait
