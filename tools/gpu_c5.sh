# BASELINE config 5 (n = 64, 2^20 problems per equation) on one GPU
for w in c5-chol c5-lyap c5-sylv; do
  timeout 900 python bench.py --workload $w --steps 5 --warmup 3 > gpurun_out/bench_$w.log 2>&1; echo "$w rc=$?"
done
