"""Wave-engine check + timing on the GPU: parity vs the CPU oracle (small
batch) and ms / GFLOP/s at the BASELINE batch against the dispatch-table
engine, per n.

    python tools/wave_check.py [--eqs lyapunov,sylvester] [--sizes 16,64,128]
"""

import argparse
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from oracle import oracle  # noqa: E402  (test infrastructure: the checker)
from paper_1906_08613_b200 import dispatch, executor  # noqa: E402
from paper_1906_08613_b200.variants import builtin_variants, default_blocks  # noqa: E402

RIGHT = {"lyapunov": 5, "sylvester": 13}


def timeit(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--eqs", default="lyapunov,sylvester")
    ap.add_argument("--sizes", default=",".join(str(n) for n in range(8, 129, 4)))
    ap.add_argument("--no-time", action="store_true")
    ap.add_argument("--no-base", action="store_true")
    args = ap.parse_args()
    torch.cuda.set_device(0)
    out = []
    for eq in args.eqs.split(","):
        v = RIGHT[eq]
        for n in [int(x) for x in args.sizes.split(",")]:
            b = default_blocks(n)[0]
            ins = executor.generate(eq, n, seed=n, batch=40)
            X, info = executor.solve(eq, ins, variant=v, b=b, engine="wave", check=False)
            host = [t.cpu().numpy() for t in ins]
            want, winfo = oracle.execute(eq, builtin_variants(eq)[v].statements, n, b, host)
            got = X.cpu().numpy()
            err = float((np.linalg.norm((got - want).reshape(40, -1), axis=1)
                         / np.maximum(1.0, np.linalg.norm(want.reshape(40, -1), axis=1))).max())
            res = float(oracle.residual(eq, n, host, got).max() / (n * np.finfo(np.float64).eps))
            sym = bool(np.array_equal(got, np.transpose(got, (0, 2, 1)))) if eq == "lyapunov" else True
            rec = {"eq": eq, "n": n, "err": err, "res_over_neps": res, "info": int(np.abs(info.cpu().numpy()).sum()),
                   "sym": sym}
            if not args.no_time:
                batch = (1 << 28) // (8 * n * n)
                big = executor.generate(eq, n, seed=n, batch=batch)
                Xb = torch.empty_like(big[-1])
                ib = torch.empty(batch, dtype=torch.int32, device="cuda")
                ms = timeit(lambda: executor.solve(eq, big, variant=v, b=b, engine="wave", out=Xb, info=ib,
                                                   check=False))
                flops = 2.0 * n ** 3 * batch
                rec.update(ms=round(ms, 4), gflops=round(flops / ms / 1e6, 1))
                if not args.no_base:
                    pick = dispatch.select(eq, n)
                    msb = timeit(lambda: executor.solve(eq, big, variant=pick["variant"], b=pick["b"],
                                                        engine=pick.get("engine", "auto"), out=Xb, info=ib,
                                                        check=False), reps=2)
                    rec.update(base_ms=round(msb, 4), base=f"{pick.get('engine')} v{pick['variant']} b{pick['b']}")
                del big, Xb, ib
            print(json.dumps(rec), flush=True)
            out.append(rec)
    bad = [r for r in out if not (r["err"] <= 1e-10 and r["res_over_neps"] <= 10 and r["info"] == 0 and r["sym"])]
    print("FAILED" if bad else "ALL OK", len(bad))


if __name__ == "__main__":
    main()
