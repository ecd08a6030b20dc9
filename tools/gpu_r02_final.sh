# Round-2 final evidence on one B200: GPU parity suite, smoke, the bench line
# (+ per-n detail), the reference arm, config 1 and config 5 lines, then the
# ncu launch lists and ncu --set full captures (tools/evidence.sh re-runs the
# bench first: each ncu command runs only after the same command exited 0).
set -u
O=gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/gpuinfo.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
tail -3 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/smoke.log
tail -2 $O/smoke.log
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_reference.log 2>&1; echo "reference arm rc=$?"
bash tools/evidence.sh
for w in c1 c5-chol c5-lyap c5-sylv; do
  timeout 900 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu > $O/bench_$w.log 2>&1; echo "$w rc=$?"
done
for eq in cholesky lyapunov sylvester; do timeout 300 python tools/e2e_probe4.py $eq; done > $O/e2e_hybrid.txt 2>&1; echo "e2e probe rc=$?"
LAGEN_HOST_SPLIT=0 timeout 300 python tools/e2e_probe4.py cholesky > $O/e2e_nosplit.txt 2>&1
