"""`mode="cuda"` generate-verify-benchmark-select pipeline: the reference's
`run_pipeline` (/root/reference/pkg/src/lagen/cli.py:184-251) with the
variant executed by the B200 library instead of emitted C.

Same steps and report schema as the reference:
  * variant space  = algorithm x admissible b (cli.py:89-120, tiles = b);
    ids `a<alg>_b<b>_t<b>_cuda` (cli.py:83-86 with the mode suffix);
  * verify         = equation residual ||lhs - rhs||_F / max(1, ||rhs||_F)
                     (verify.py:186-195) of every problem of a seeded batch
                     at every size, against `tol` (cli.py:131-143);
  * benchmark      = median device time of the batched launch (CUDA events
                     on the launching stream) -> `median_ns` per problem, and
                     one `RESULT <id> <n> <median_ns> <flops>` line per row
                     (the harness line, codegen.py:496-578);
  * select         = fastest median, ties on flops then id (cli.py:175-181).
Rows carry `"mode": "cuda"` and, beside the reference's fields, the batch,
the batched median in ms and the engine the dispatch used.

    python -m paper_1906_08613_b200.pipeline --eq cholesky --sizes 16,32
"""

import argparse
import json
import statistics
import sys
from dataclasses import dataclass

import torch

from . import dispatch, errors, executor
from .variants import EQUATIONS, builtin_variants, default_blocks, flop_count

# With the reference importable its own pieces are used, not restated: the
# selection rule `_select` (cli.py:175-181), the admissible blocks
# (cli.py:89-93), and — for live Equation objects, run_pipeline_live below —
# its variant enumeration, instances, residual and flop model.
try:  # pragma: no cover - depends on the environment
    from lagen import cli as _ref_cli
except Exception:  # the GPU box has no reference package
    _ref_cli = None

DEFAULT_SEED = 0
DEFAULT_TOL = 1e-10  # cli.py DEFAULT_TOL, the harness GUARD (codegen.py:496-578)
DEFAULT_REPS = 5


@dataclass(frozen=True)
class CudaVariantConfig:
    """VariantConfig (cli.py:68-86) with mode "cuda": tiles = b, no nu."""
    algorithm_index: int
    b: int
    mode: str = "cuda"

    @property
    def tiles(self):
        return self.b

    @property
    def id(self):
        return f"a{self.algorithm_index}_b{self.b}_t{self.b}_cuda"


def _eq_name(eq):
    name = getattr(eq, "name", eq)
    if name not in EQUATIONS:
        raise errors.UsageError(f"unknown equation {eq!r}")
    return name


def enumerate_variants(eq, n, blocks=None):
    """Cross product of the built-in algorithms x admissible block sizes
    (cli.py:95-120; `blocks` filtered to b <= n, b | n like the reference)."""
    eq = _eq_name(eq)
    if n < 2:
        raise errors.UsageError("n must be at least 2")
    if blocks is None:
        blocks = default_blocks(n)
    blocks = [b for b in blocks if b <= n and n % b == 0]
    if not blocks:
        raise errors.UsageError(f"no admissible block size divides n={n}")
    out = [CudaVariantConfig(v.index, b) for v in builtin_variants(eq) for b in blocks]
    if not out:
        raise errors.UsageError("variant search space is empty")
    return out


def residuals_device(eq, inputs, X):
    """Per-problem ||lhs - rhs||_F / max(1, ||rhs||_F) on the device
    (verify.py:186-195) for a batch: chol X^T X = A, lyap L X + X L^T = S,
    sylv L X + X U = C."""
    eq = _eq_name(eq)
    if eq == "cholesky":
        (A,) = inputs
        lhs, rhs = torch.bmm(X.transpose(1, 2), X), A
    elif eq == "lyapunov":
        L, S = inputs
        lhs, rhs = torch.bmm(L, X) + torch.bmm(X, L.transpose(1, 2)), S
    else:
        L, U, C = inputs
        lhs, rhs = torch.bmm(L, X) + torch.bmm(X, U), C
    num = torch.linalg.matrix_norm(lhs - rhs)
    den = torch.clamp(torch.linalg.matrix_norm(rhs), min=1.0)
    return num / den


def verify_variant(eq, cfg, sizes, seed=DEFAULT_SEED, tol=DEFAULT_TOL, batch=64):
    """Residuals of the variant at every size (cli.py:131-143): the worst
    problem of a seeded batch per size; None where b does not divide n."""
    eq = _eq_name(eq)
    out = {}
    for n in sizes:
        if n % cfg.b:
            out[str(n)] = None
            continue
        ins = executor.generate(eq, n, seed=seed + n, batch=batch)
        X, info = executor.solve(eq, ins, variant=cfg.algorithm_index, b=cfg.b, check=False)
        bad = bool((info != 0).any())
        r = float(residuals_device(eq, ins, X).max())
        out[str(n)] = float("inf") if bad else r
    checked = [r for r in out.values() if r is not None]
    return out, bool(checked) and all(r <= tol for r in checked)


def benchmark_variant(eq, cfg, n, batch=None, reps=DEFAULT_REPS, seed=DEFAULT_SEED):
    """Median device time of `reps` batched launches (one warm-up); returns
    (median ns per problem, median ms per batch, batch, engine)."""
    eq = _eq_name(eq)
    if batch is None:
        batch = max(1, (1 << 28) // (8 * n * n))
    ins = executor.generate(eq, n, seed=seed + n, batch=batch)
    # a live reference Algorithm (run_pipeline_live) is encoded by the executor
    plan = executor.Plan(eq, ins, variant=getattr(cfg, "algorithm", None) or cfg.algorithm_index, b=cfg.b)
    stream = torch.cuda.current_stream()
    plan.launch(stream)
    ts = []
    for _ in range(reps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(stream)
        plan.launch(stream)
        e.record(stream)
        e.synchronize()
        ts.append(s.elapsed_time(e))
    ms = statistics.median(ts)
    return int(round(ms * 1e6 / batch)), ms, batch, plan.engine


def _select(rows):
    """Mark the fastest verified row; ties break on flops, then id
    (cli.py:175-181; the reference's own function when importable)."""
    if _ref_cli is not None:
        return _ref_cli._select(rows)
    timed = [r for r in rows if r["median_ns"] is not None]
    if not timed:
        return
    best = min(timed, key=lambda r: (r["median_ns"], r["flops"], r["id"]))
    best["selected"] = True


def run_pipeline(eq, sizes, seed=DEFAULT_SEED, tol=DEFAULT_TOL, blocks=None, reps=DEFAULT_REPS,
                 batch=None, benchmark=True, log=print):
    """Generate -> verify -> benchmark -> select for one equation at
    max(sizes) (cli.py:184-251).  Returns (report, all_verified,
    benchmark_failures) with the reference's report schema."""
    eq = _eq_name(eq)
    target_n = max(sizes)
    rows = []
    for cfg in enumerate_variants(eq, target_n, blocks):
        residuals, passed = verify_variant(eq, cfg, sizes, seed, tol)
        alg = builtin_variants(eq)[cfg.algorithm_index]
        rows.append({
            "id": cfg.id,
            "algorithm": cfg.algorithm_index,
            "invariant": alg.invariant,
            "b": cfg.b,
            "tiles": cfg.tiles,
            "mode": "cuda",
            "flops": flop_count(eq, alg.statements, target_n, cfg.b),
            "residuals": residuals,
            "median_ns": None,
            "selected": False,
            "verified": passed,
        })
    failures = 0
    if benchmark:
        for row in rows:
            if not row["verified"]:
                continue
            cfg = CudaVariantConfig(row["algorithm"], row["b"])
            try:
                ns, ms, nb, engine = benchmark_variant(eq, cfg, target_n, batch, reps, seed)
            except errors.LagenError as err:
                failures += 1
                log(f"benchmark {row['id']}: {err}", file=sys.stderr)
                continue
            row.update(median_ns=ns, batch=nb, median_ms=ms, engine=engine)
            log(f"RESULT {row['id']} {target_n} {ns} {row['flops']}")
        _select(rows)
    all_verified = all(r["verified"] for r in rows)
    for row in rows:
        del row["verified"]
    return {"equation": eq, "n": target_n, "variants": rows}, all_verified, failures


def live_variant_configs(eq, n, blocks=None):
    """The reference's own variant space for a live `Equation`
    (cli.enumerate_variants, cli.py:95-120: its synthesised `Algorithm`
    objects x admissible b, tiles = b) re-tagged mode "cuda": each config is a
    reference `VariantConfig` subclass instance whose id ends in `_cuda`."""
    if _ref_cli is None:
        raise errors.UsageError("the reference package `lagen` is not importable")

    class CudaConfig(_ref_cli.VariantConfig):
        @property
        def id(self):
            return f"a{self.algorithm_index}_b{self.b}_t{self.tiles}_cuda"

    return [CudaConfig(c.algorithm, c.algorithm_index, c.b, c.tiles, "cuda")
            for c in _ref_cli.enumerate_variants(eq, n, blocks, None, "scalar")]


def run_pipeline_live(eq, sizes, seed=DEFAULT_SEED, tol=DEFAULT_TOL, blocks=None, reps=DEFAULT_REPS,
                      batch=None, benchmark=True, log=print):
    """`run_pipeline` (cli.py:184-251) driven by the reference's own objects:
    `eq` is a live `lagen` Equation; the variant space, the verification
    instances (`random_instance`), the residual, the flop model, the report
    schema and `_select` are the reference's — only the two execution steps
    are replaced: `interpret_algorithm` -> executor.interpret_algorithm (the
    CUDA kernel run from the live Algorithm's statements) and the emitted-C
    harness -> benchmark_variant above."""
    from lagen import verify as rverify
    from lagen.worksheet import flop_count as ref_flop_count

    target_n = max(sizes)
    rows, cfgs = [], {}
    for cfg in live_variant_configs(eq, target_n, blocks):
        residuals = {}
        for n in sizes:
            if n % cfg.b:
                residuals[str(n)] = None
                continue
            inst = rverify.random_instance(cfg.algorithm.equation, n, seed)
            try:
                outputs, _ = executor.interpret_algorithm(cfg.algorithm, inst, cfg.b)
                residuals[str(n)] = float(rverify.residual(cfg.algorithm.equation, inst, outputs))
            except errors.VerificationError:
                residuals[str(n)] = float("inf")
        checked = [r for r in residuals.values() if r is not None]
        cfgs[cfg.id] = cfg
        rows.append({
            "id": cfg.id,
            "algorithm": cfg.algorithm_index,
            "invariant": cfg.algorithm.invariant.label(),
            "b": cfg.b,
            "tiles": cfg.tiles,
            "mode": "cuda",
            "flops": ref_flop_count(cfg.algorithm, target_n, cfg.b),
            "residuals": residuals,
            "median_ns": None,
            "selected": False,
            "verified": bool(checked) and all(r <= tol for r in checked),
        })
    failures = 0
    if benchmark:
        for row in rows:
            if not row["verified"]:
                continue
            try:
                ns, ms, nb, engine = benchmark_variant(eq.name, cfgs[row["id"]], target_n, batch, reps, seed)
            except errors.LagenError as err:
                failures += 1
                log(f"benchmark {row['id']}: {err}", file=sys.stderr)
                continue
            row.update(median_ns=ns, batch=nb, median_ms=ms, engine=engine)
            log(f"RESULT {row['id']} {target_n} {ns} {row['flops']}")
        _select(rows)
    all_verified = all(r["verified"] for r in rows)
    for row in rows:
        del row["verified"]
    return {"equation": eq.name, "n": target_n, "variants": rows}, all_verified, failures


def selected(report):
    """(variant, b) of the selected row, or None."""
    for r in report["variants"]:
        if r["selected"]:
            return r["algorithm"], r["b"]
    return None


def main(argv=None):
    ap = argparse.ArgumentParser(description=__doc__.splitlines()[0])
    ap.add_argument("--eq", required=True, choices=EQUATIONS)
    ap.add_argument("--sizes", required=True, help="comma-separated n; benchmark at max")
    ap.add_argument("--blocks", default=None)
    ap.add_argument("--seed", type=int, default=DEFAULT_SEED)
    ap.add_argument("--tol", type=float, default=DEFAULT_TOL)
    ap.add_argument("--reps", type=int, default=DEFAULT_REPS)
    ap.add_argument("--batch", type=int, default=None)
    ap.add_argument("--no-bench", action="store_true")
    a = ap.parse_args(argv)
    sizes = [int(x) for x in a.sizes.split(",") if x]
    blocks = [int(x) for x in a.blocks.split(",")] if a.blocks else None
    report, ok, fails = run_pipeline(a.eq, sizes, a.seed, a.tol, blocks, a.reps, a.batch, not a.no_bench)
    print(json.dumps(report, indent=1))
    if not ok:
        return 1  # cli.py:385-406: verification failure -> exit 1
    return 2 if fails else 0


if __name__ == "__main__":
    sys.exit(main())
