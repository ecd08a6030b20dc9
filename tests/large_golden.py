"""Helpers for the large-n reference goldens (tests/golden/make_golden_large.py):
regenerate the inputs with the oracle's CPU generator, check them against the
stored checksums, and compare an output batch's projections with the
reference's."""

import json
from pathlib import Path

import numpy as np

GOLDEN = Path(__file__).resolve().parent / "golden"
META = json.loads((GOLDEN / "large_meta.json").read_text())


def projectors(n):
    rng = np.random.default_rng(1000 + n)
    return rng.standard_normal((n, 2)), rng.standard_normal((n, 2))


def data(eq):
    return np.load(GOLDEN / f"large_{eq}.npz")


def inputs(oracle_mod, eq, n, d):
    """The NPROB problems the goldens were made from (checksums verified)."""
    gen = oracle_mod.generate(eq, n, seed=n, first=0, batch=META["nprob"])
    got = [float(np.sum(a)) for a in gen] + [float(np.sum(a * a)) for a in gen]
    want = d[f"checksum_{n}"]
    assert np.allclose(got, want, rtol=1e-12, atol=0), (eq, n, "generator drifted from the golden inputs")
    return gen


def groups(eq):
    """{(n, variant, b): [entries ordered by problem]}"""
    out = {}
    for e in META[eq]:
        out.setdefault((e["n"], e["variant"], e["b"]), []).append(e)
    for v in out.values():
        v.sort(key=lambda e: e["p"])
    return out


def max_rel_err(X, d, entries):
    """max over problems of the projection errors, relative to
    ||X_ref||_F * ||V||_F (a bound implied by ||X - X_ref|| <= tol ||X_ref||)."""
    n = X.shape[1]
    V, W = projectors(n)
    worst = 0.0
    for e in entries:
        k = e["key"]
        x = X[e["p"]]
        nrm = max(1.0, float(d["nrm_" + k][0]))
        e1 = np.linalg.norm(x @ V - d["xv_" + k]) / (nrm * np.linalg.norm(V))
        e2 = np.linalg.norm(W.T @ x - d["wx_" + k]) / (nrm * np.linalg.norm(W))
        worst = max(worst, e1, e2)
    return worst
