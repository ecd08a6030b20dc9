"""GPU autotuner: time every (variant, b) per (equation, n) on a B200 and
write the dispatch table — the GPU analogue of `lagen tune`'s empirical
selection (/root/reference/pkg/src/lagen/cli.py:146-181: fastest median,
ties broken by flops then id; here flops are variant-independent).

    python tools/autotune.py [--sizes 4,8,...] [--eqs cholesky,...] [--reps 5]

Writes paper_1906_08613_b200/dispatch_table.json and a full report to
gpurun_out/autotune_report.json.  Inputs: BASELINE batch floor(2^28/8n^2)
(>= L2) from the seeded generator; every candidate is checked against the
first candidate's output (<= 1e-10) before it may win.
"""

import argparse
import json
import statistics
import sys
from pathlib import Path

import torch

REPO = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(REPO))

from paper_1906_08613_b200 import executor  # noqa: E402
from paper_1906_08613_b200.variants import EQUATIONS, builtin_variants, default_blocks  # noqa: E402


def _lib_eq(eq):
    return EQUATIONS.index(eq)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default=",".join(str(n) for n in range(4, 129, 4)))
    ap.add_argument("--eqs", default=",".join(EQUATIONS))
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--engines", default="all")
    ap.add_argument("--merge", action="store_true",
                    help="keep an existing table entry unless a timed candidate beats its ms")
    ap.add_argument("--out", default=str(REPO / "paper_1906_08613_b200" / "dispatch_table.json"))
    ap.add_argument("--report", default=str(REPO / "gpurun_out" / "autotune_report.json"))
    args = ap.parse_args()
    torch.cuda.set_device(0)
    sizes = [int(x) for x in args.sizes.split(",")]
    table = json.loads(Path(args.out).read_text()) if Path(args.out).exists() else {}
    report = {}
    stream = torch.cuda.Stream()
    for eq in args.eqs.split(","):
        table.setdefault(eq, {})
        report[eq] = {}
        for n in sizes:
            batch = (1 << 28) // (8 * n * n)
            with torch.cuda.stream(stream):
                ins = executor.generate(eq, n, seed=n, batch=batch, stream=stream)
            stream.synchronize()
            rows = []
            ref_X = None
            from paper_1906_08613_b200 import _lib
            # the reference's default blocks plus b = n (admissible: verify.py:232-233)
            blocks = sorted(set(default_blocks(n)) | {n})
            cands = [(v, b, e) for e in ("generic", "warp", "column", "dataflow", "rows", "wave", "rowspad",
                                         "pipe", "rowsweep", "rowsmix")
                     for v in builtin_variants(eq) for b in blocks
                     if _lib.engine_supported(_lib_eq(eq), n, b, v.index, e)
                     # rowsweep runs the same kernel for every variant (b = n): time one
                     and not (e == "rowsweep" and v.index != {"lyapunov": 5, "sylvester": 13}.get(eq))]
            if args.engines != "all":
                cands = [c for c in cands if c[2] in args.engines.split(",")]
            for v, b, engine in cands:
                if True:
                    plan = executor.Plan(eq, ins, variant=v.index, b=b, engine=engine)
                    with torch.cuda.stream(stream):
                        plan.launch(stream)
                        plan.launch(stream)
                    stream.synchronize()
                    ok = bool((plan.info == 0).all())
                    if ref_X is None:
                        ref_X = plan.out.clone()
                    else:
                        d = torch.linalg.matrix_norm(plan.out - ref_X) / torch.clamp(
                            torch.linalg.matrix_norm(ref_X), min=1.0)
                        ok = ok and float(d.max()) <= 1e-10
                    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                           for _ in range(args.reps)]
                    with torch.cuda.stream(stream):
                        for a, e in evs:
                            a.record(stream)
                            plan.launch(stream)
                            e.record(stream)
                    stream.synchronize()
                    ms = statistics.median(a.elapsed_time(e) for a, e in evs)
                    rows.append({"variant": v.index, "b": b, "engine": engine, "ms": round(ms, 5), "ok": ok})
                    del plan
            good = [r for r in rows if r["ok"]]
            if not good:
                continue
            best = min(good, key=lambda r: (r["ms"], r["variant"], r["b"]))
            old = table[eq].get(str(n))
            if args.merge and old is not None and old.get("ms", 1e30) <= best["ms"]:
                print(f"{eq} n={n}: keep {old} (candidate {best['engine']} {best['ms']:.4f} ms)", flush=True)
                report[eq][str(n)] = rows
                continue
            table[eq][str(n)] = {"variant": best["variant"], "b": best["b"], "engine": best["engine"],
                                 "ms": best["ms"]}
            report[eq][str(n)] = rows
            print(f"{eq} n={n}: best v{best['variant']} b{best['b']} {best['engine']} {best['ms']:.4f} ms "
                  f"(worst {max(r['ms'] for r in rows):.4f} ms)", flush=True)
            del ins, ref_X
            torch.cuda.empty_cache()
    Path(args.out).write_text(json.dumps(table, indent=1) + "\n")
    Path(args.report).parent.mkdir(exist_ok=True)
    (Path(args.report).parent / "dispatch_table.json").write_text(json.dumps(table, indent=1) + "\n")
    Path(args.report).parent.mkdir(exist_ok=True)
    Path(args.report).write_text(json.dumps(report, indent=1) + "\n")


if __name__ == "__main__":
    main()
