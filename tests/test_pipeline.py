"""mode="cuda" pipeline (paper_1906_08613_b200/pipeline.py) — the reference's
run_pipeline / _select (cli.py:175-251) with the B200 executor."""

import pytest

from paper_1906_08613_b200 import errors, pipeline
from paper_1906_08613_b200.variants import builtin_variants, default_blocks


def test_variant_space_matches_reference_enumeration():
    # cli.py:95-120: algorithms x admissible b (b <= n, b | n), tiles = b
    for eq, nalg in (("cholesky", 3), ("lyapunov", 6), ("sylvester", 14)):
        for n in (4, 16, 24, 32):
            vs = pipeline.enumerate_variants(eq, n)
            assert len(vs) == nalg * len(default_blocks(n))
            assert {v.algorithm_index for v in vs} == {v.index for v in builtin_variants(eq)}
            assert all(v.id == f"a{v.algorithm_index}_b{v.b}_t{v.b}_cuda" for v in vs)
    assert [v.b for v in pipeline.enumerate_variants("cholesky", 12, blocks=[3, 4, 5, 24])] == [3, 4] * 3
    with pytest.raises(errors.UsageError):
        pipeline.enumerate_variants("cholesky", 7, blocks=[4])
    with pytest.raises(errors.UsageError):
        pipeline.enumerate_variants("cholesky", 1)


def test_select_rule():
    # fastest median, ties on flops, then id (cli.py:175-181); untimed rows never win
    rows = [{"id": "a1_b4_t4_cuda", "median_ns": 10, "flops": 5, "selected": False},
            {"id": "a0_b4_t4_cuda", "median_ns": 10, "flops": 5, "selected": False},
            {"id": "a2_b4_t4_cuda", "median_ns": 10, "flops": 4, "selected": False},
            {"id": "a3_b4_t4_cuda", "median_ns": None, "flops": 1, "selected": False}]
    pipeline._select(rows)
    assert [r["id"] for r in rows if r["selected"]] == ["a2_b4_t4_cuda"]
    rows[2]["flops"] = 5
    for r in rows:
        r["selected"] = False
    pipeline._select(rows)
    assert [r["id"] for r in rows if r["selected"]] == ["a0_b4_t4_cuda"]


@pytest.mark.gpu
@pytest.mark.parametrize("eq", ["cholesky", "lyapunov", "sylvester"])
def test_run_pipeline_cuda(eq):
    lines = []
    report, ok, fails = pipeline.run_pipeline(eq, [8, 16], reps=2, batch=256,
                                              log=lambda *a, **k: lines.append(" ".join(map(str, a))))
    assert ok and fails == 0
    assert report["equation"] == eq and report["n"] == 16
    rows = report["variants"]
    assert len(rows) == len(builtin_variants(eq)) * len(default_blocks(16))
    assert sum(r["selected"] for r in rows) == 1
    assert all(r["mode"] == "cuda" and r["median_ns"] > 0 for r in rows)
    assert all(max(v for v in r["residuals"].values() if v is not None) <= pipeline.DEFAULT_TOL for r in rows)
    res = [l.split() for l in lines if l.startswith("RESULT")]
    assert len(res) == len(rows) and all(len(p) == 5 and p[2] == "16" for p in res)
    assert pipeline.selected(report) is not None


def test_live_pipeline_uses_the_reference_objects(oracle_mod, monkeypatch):
    """run_pipeline_live on a live lagen Equation: the reference's variant
    space, instances, residual, flop model, schema and _select, with the two
    execution steps replaced (here by the CPU oracle and a fixed timing, no
    GPU) — row for row against the reference's own run_pipeline."""
    pytest.importorskip("lagen")
    import numpy as np
    from lagen import cli
    from lagen.lang import parse_equation
    from paper_1906_08613_b200 import executor
    from paper_1906_08613_b200.variants import EQ_INPUTS, encode_algorithm

    eq = parse_equation("Equation: L * X + X * L^T = S\nL: Matrix(n,n), lower_triangular, input\n"
                        "S: Matrix(n,n), symmetric, input\nX: Matrix(n,n), symmetric, output\n", name="lyapunov")

    def fake_interpret(alg, inst, b, on_iteration=None):
        ins = [np.ascontiguousarray(inst.bindings[nm], dtype=np.float64)[None] for nm in EQ_INPUTS["lyapunov"]]
        X, info = oracle_mod.execute("lyapunov", encode_algorithm(alg), inst.n, b, ins)
        assert int(info[0]) == 0
        return {alg.output: X[0]}, 0

    times = iter(range(100, 0, -1))
    monkeypatch.setattr(executor, "interpret_algorithm", fake_interpret)
    monkeypatch.setattr(pipeline, "benchmark_variant", lambda *a, **k: (next(times), 1.0, 8, "stub"))
    lines = []
    got, ok, fails = pipeline.run_pipeline_live(eq, [8, 16], log=lambda *a, **k: lines.append(a[0]))
    want, wok, _ = cli.run_pipeline(eq, [8, 16], cc=None)
    assert ok and wok and fails == 0
    assert got["equation"] == want["equation"] and got["n"] == want["n"]
    assert len(got["variants"]) == len(want["variants"])
    for g, w in zip(got["variants"], want["variants"]):
        assert g["id"] == w["id"].replace("_scalar", "_cuda") and g["mode"] == "cuda"
        for k in ("algorithm", "invariant", "b", "tiles", "flops"):
            assert g[k] == w[k]
        assert set(g["residuals"]) == set(w["residuals"])
        assert all(r is None or r <= 1e-10 for r in g["residuals"].values())
    # the reference's own _select ran on the rows: the last (fastest stub time) wins
    assert [r["selected"] for r in got["variants"]] == [False] * (len(got["variants"]) - 1) + [True]
    assert pipeline._select.__doc__ and pipeline._ref_cli is cli
    assert len(lines) == len(got["variants"]) and all(l.startswith("RESULT a") for l in lines)
