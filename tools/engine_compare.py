"""Compare engines on one equation: parity against the first engine listed and
device time per batched solve (full-HBM batch).

    python tools/engine_compare.py --eq sylvester --sizes 32,64,124,128 \
        --runs 13:4:warp,13:4:dataflow
"""
import argparse
import json
import sys
from pathlib import Path

import torch

import os  # noqa: E402
sys.path.insert(0, os.environ.get("LAGEN_PKG_ROOT", str(Path(__file__).resolve().parents[1])))
from paper_1906_08613_b200 import _lib, executor  # noqa: E402
from paper_1906_08613_b200.variants import EQ_CODES  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--eq", default="sylvester")
ap.add_argument("--sizes", default="32,64,128")
ap.add_argument("--runs", default="13:4:warp,13:4:dataflow", help="variant:b:engine,...")
ap.add_argument("--bytes", type=float, default=2 ** 28)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--json", default=None)
a = ap.parse_args()
torch.cuda.set_device(0)
out = []
for n in [int(x) for x in a.sizes.split(",")]:
    batch = max(1, int(a.bytes // (8 * n * n)))
    ins = executor.generate(a.eq, n, seed=n, batch=batch)
    ref = None
    for r in a.runs.split(","):
        v, b, eng = r.split(":")
        v, b = int(v), int(b)
        b = b or n  # 0: b = n
        if n % b or not _lib.engine_supported(EQ_CODES[a.eq], n, b, v, eng):
            continue
        plan = executor.Plan(a.eq, ins, variant=v, b=b, engine=eng)
        plan.launch()
        torch.cuda.synchronize()
        bad = int((plan.info != 0).sum())
        if ref is None:
            ref = plan.out.clone()
            err = 0.0
        else:
            d = torch.linalg.matrix_norm(plan.out - ref) / torch.clamp(torch.linalg.matrix_norm(ref), min=1.0)
            err = float(d.max())
        ts = []
        for _ in range(a.reps):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            plan.launch()
            e.record()
            torch.cuda.synchronize()
            ts.append(s.elapsed_time(e))
        ms = min(ts)
        rec = dict(eq=a.eq, n=n, variant=v, b=b, engine=eng, batch=batch, ms=ms, us_per_kprob=1e3 * ms / batch * 1e3,
                   err=err, info_nonzero=bad)
        out.append(rec)
        print(json.dumps(rec), flush=True)
if a.json:
    Path(a.json).write_text(json.dumps(out, indent=1))
