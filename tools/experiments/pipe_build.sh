#!/bin/bash
# tools/experiments/pipe_build.sh "EQ N MODE [tag] [extra flags]" ... -> tools/experiments/pipe_bin/p_EQ_N_MODE_tag
mkdir -p tools/experiments/pipe_bin
for cfg in "$@"; do
  set -- $cfg
  eq=$1; n=$2; mode=$3; tag=${4:-base}; if [ $# -ge 4 ]; then shift 4; else shift 3; fi
  out=tools/experiments/pipe_bin/p_${eq}_${n}_${mode}_${tag}
  nvcc -cudart shared -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++20 --expt-relaxed-constexpr -Xptxas -v -DPEQ=$eq -DPN=$n -DPMODE=$mode ${PIPE_PROF--DLAGEN_PIPE_PROF=1} "$@" \
     -Iinclude -I${PIPE_SRC:-paper_1906_08613_b200/csrc} tools/experiments/pipe_bench.cu -o $out 2>&1 | grep -E "error|registers|spill" | grep -v "_Z3gen" | grep -v "^ptxas info    : Function" | grep -v "32 registers\|0 bytes stack" | sed "s/^/$eq $n $mode $tag: /" &
done
wait
