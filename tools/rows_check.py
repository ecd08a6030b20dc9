"""Cholesky rows-engine check: per size, device time of one
full-HBM batched solve (b = 8 kernel; n = 4 mod 8 through the padded
instance) and the max relative difference to the CPU oracle on a sample.

    python tools/rows_check.py --sizes 40,64,128
"""
import argparse, json, os, sys
from pathlib import Path
import numpy as np
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle import oracle  # noqa: E402  (checker only)
from paper_1906_08613_b200 import executor  # noqa: E402
from paper_1906_08613_b200.variants import builtin_variants  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--sizes", default="40,64,96,128")
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--sample", type=int, default=48)
a = ap.parse_args()
torch.cuda.set_device(0)
stm = builtin_variants("cholesky")[1].statements
for n in [int(x) for x in a.sizes.split(",")]:
    batch = (1 << 28) // (8 * n * n)
    ins = executor.generate("cholesky", n, seed=n, batch=batch)
    if n % 8 == 0:
        plan = executor.Plan("cholesky", ins, variant=1, b=8, engine="rows")
    else:
        plan = executor.Plan("cholesky", ins, variant=1, b=4, engine="rowspad")
    plan.launch()
    torch.cuda.synchronize()
    ts = []
    for _ in range(a.reps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); plan.launch(); e.record(); torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    idx = np.linspace(0, batch - 1, a.sample).astype(np.int64)
    host = [t[idx].cpu().numpy() for t in ins]
    want, winfo = oracle.execute("cholesky", stm, n, 4, host)
    got = plan.out[idx].cpu().numpy()
    err = np.linalg.norm((got - want).reshape(len(idx), -1), axis=1) / np.maximum(
        1.0, np.linalg.norm(want.reshape(len(idx), -1), axis=1))
    print(json.dumps(dict(n=n, ms=min(ts), batch=batch,
                          err=float(err.max()), info_nonzero=int((plan.info != 0).sum()))), flush=True)
