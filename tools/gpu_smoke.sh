# round-end style checks: smoke(), BASELINE configs[0] line, reference arm line
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py --workload c1 --steps 10 --warmup 3 > gpurun_out/bench_c1.log 2>&1; echo "c1 rc=$?"
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?"
