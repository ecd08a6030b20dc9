"""Run one batched solve configuration a few times (ncu / debugging target)."""
import argparse, sys
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1906_08613_b200 import executor

ap = argparse.ArgumentParser()
ap.add_argument("--eq", default="cholesky")
ap.add_argument("--n", type=int, default=64)
ap.add_argument("--b", type=int, default=None)
ap.add_argument("--variant", type=int, default=None)
ap.add_argument("--batch", type=int, default=None)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--engine", default=None)
a = ap.parse_args()
torch.cuda.set_device(0)
batch = a.batch or (1 << 28) // (8 * a.n * a.n)
ins = executor.generate(a.eq, a.n, seed=a.n, batch=batch)
plan = executor.Plan(a.eq, ins, variant=a.variant, b=a.b, engine=a.engine)
for _ in range(a.reps):
    plan.launch()
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record(); plan.launch(); e.record(); torch.cuda.synchronize()
print(f"{a.eq} n={a.n} v{plan.variant} b{plan.b} batch={batch} {s.elapsed_time(e):.4f} ms, info_nonzero={int((plan.info!=0).sum())}")
