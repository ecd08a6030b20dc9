"""Pin the CPU oracle (oracle/lagen_oracle.c) to the reference.

Golden vectors come from the reference's own executor
(interpret_algorithm, verify.py:221-303) via tests/golden/make_golden.py;
the known-answer tests restate pkg/tests/test_verify.py.  CPU only.
"""

import json
from pathlib import Path

import numpy as np
import pytest

from paper_1906_08613_b200.variants import (EQ_INPUTS, EQUATIONS, builtin_variants,
                                             bytes_compulsory, flop_count, flops_alg)

GOLDEN = Path(__file__).resolve().parent / "golden"
META = json.loads((GOLDEN / "golden_meta.json").read_text())


def _golden(eq):
    return np.load(GOLDEN / f"{eq}.npz")


@pytest.mark.parametrize("eq", EQUATIONS)
def test_oracle_matches_reference_interpreter(eq, oracle_mod):
    """Every variant x b x n in the fixture, two instance families, <= 1e-13."""
    d = _golden(eq)
    vs = builtin_variants(eq)
    worst = 0.0
    for e in META[eq]["entries"]:
        ins = [d[f"in_{e['case']}_{e['n']}_{nm}"][None] for nm in EQ_INPUTS[eq]]
        X, info = oracle_mod.execute(eq, vs[e["variant"]].statements, e["n"], e["b"], ins)
        want = d[e["key"]]
        assert info[0] == 0
        err = np.linalg.norm(X[0] - want) / max(1.0, np.linalg.norm(want))
        worst = max(worst, err)
    assert worst <= 1e-13, worst


@pytest.mark.parametrize("eq", EQUATIONS)
def test_golden_flop_counts_match_model(eq):
    """The reference's dynamic counter equals the restated flop model."""
    vs = builtin_variants(eq)
    for e in META[eq]["entries"]:
        assert flop_count(eq, vs[e["variant"]].statements, e["n"], e["b"]) == e["flops"]
        assert e["flops"] == flops_alg(eq, e["n"])


def test_flop_totals_at_32():
    # pkg/test_output.txt:212
    assert flops_alg("cholesky", 32) == 11440
    assert flops_alg("sylvester", 32) == 65536
    assert flops_alg("lyapunov", 32) == 33792
    # unblocked Cholesky n = 4 -> 30 flops (pkg/tests/test_verify.py:144-152)
    assert flop_count("cholesky", builtin_variants("cholesky")[0].statements, 4, 4) == 30


@pytest.mark.parametrize("eq", EQUATIONS)
def test_oracle_vs_independent_oracle(eq, oracle_mod):
    """Against verify.oracle_solve outputs (textbook / Kronecker), n <= 16."""
    d = _golden(eq)
    vs = builtin_variants(eq)
    for e in META[eq]["entries"]:
        if e["n"] > 16:
            continue
        ins = [d[f"in_{e['case']}_{e['n']}_{nm}"][None] for nm in EQ_INPUTS[eq]]
        X, _ = oracle_mod.execute(eq, vs[e["variant"]].statements, e["n"], e["b"], ins)
        want = d[f"oracle_{e['case']}_{e['n']}"]
        assert np.linalg.norm(X[0] - want) <= 1e-10 * max(1.0, np.linalg.norm(want))


def test_cholesky_of_identity(oracle_mod):
    for n in (4, 8):
        for v in builtin_variants("cholesky"):
            X, info = oracle_mod.execute("cholesky", v.statements, n, 4, [np.eye(n)[None]])
            assert info[0] == 0 and np.array_equal(X[0], np.eye(n))


def test_two_by_two_sylvester_kronecker_fixture(oracle_mod):
    # pkg/tests/test_verify.py:74-85
    l = np.array([[1.0, 0.0], [1.0, 2.0]])
    u = np.array([[1.0, 1.0], [0.0, 3.0]])
    c = np.ones((2, 2))
    want = oracle_mod.kron_solve(l, u, c)
    for v in builtin_variants("sylvester"):
        for b in (1, 2):
            X, _ = oracle_mod.execute("sylvester", v.statements, 2, b, [l[None], u[None], c[None]])
            assert np.allclose(X[0], want, atol=1e-14)
            assert np.max(np.abs(l @ X[0] + X[0] @ u - c)) <= 1e-14


def test_scalar_sylvester_closed_form(oracle_mod):
    # pkg/tests/test_verify.py:65-71: L = 2, U = 3, C = 10 -> X = 2
    v = builtin_variants("sylvester")[13]
    X, _ = oracle_mod.execute("sylvester", v.statements, 1, 1,
                              [np.full((1, 1, 1), 2.0), np.full((1, 1, 1), 3.0), np.full((1, 1, 1), 10.0)])
    assert X[0, 0, 0] == pytest.approx(2.0)


def test_textbook_cholesky_and_non_spd(oracle_mod):
    g = oracle_mod.generate("cholesky", 16, seed=3, first=0, batch=4)
    X, info = oracle_mod.chol_textbook(g[0])
    assert (info == 0).all()
    for v in builtin_variants("cholesky"):
        Y, info2 = oracle_mod.execute("cholesky", v.statements, 16, 4, g)
        assert (info2 == 0).all()
        assert np.abs(X - Y).max() <= 1e-12 * np.abs(X).max()
    A = g[0].copy()
    A[1, 5, 5] = -50.0  # pivot 5 becomes non-positive
    _, info3 = oracle_mod.execute("cholesky", builtin_variants("cholesky")[2].statements, 16, 4, [A])
    assert info3[0] == 0 and info3[1] == 6


@pytest.mark.parametrize("eq", EQUATIONS)
def test_generator_distributions(eq, oracle_mod):
    n = 16
    outs = oracle_mod.generate(eq, n, seed=5, first=0, batch=64)
    if eq == "cholesky":
        A = outs[0]
        assert np.array_equal(A, np.transpose(A, (0, 2, 1)))
        assert np.all(np.linalg.eigvalsh(A) > 0)
        assert abs(np.mean(np.diagonal(A, axis1=1, axis2=2)) - 2 * n) < 2.0  # E[diag] = n + n
    else:
        L = outs[0]
        assert np.all(np.triu(L, 1) == 0)
        d = np.diagonal(L, axis1=1, axis2=2)
        assert d.min() >= 1.0 and d.max() <= 2.0
        off = L[:, np.tril_indices(n, -1)[0], np.tril_indices(n, -1)[1]] * n
        assert abs(off.mean()) < 0.1 and abs(off.std() - 1.0) < 0.1
        if eq == "lyapunov":
            S = outs[1]
            assert np.array_equal(S, np.transpose(S, (0, 2, 1)))
        else:
            assert np.all(np.tril(outs[1], -1) == 0)
            C = outs[2]
            assert abs(C.mean()) < 0.05 and abs(C.std() - 1.0) < 0.05


def test_generator_shard_invariance(oracle_mod):
    """Problem p depends only on (eq, n, seed, p): any split gives the same data."""
    whole = oracle_mod.generate("sylvester", 8, seed=7, first=0, batch=10)
    a = oracle_mod.generate("sylvester", 8, seed=7, first=0, batch=3)
    b = oracle_mod.generate("sylvester", 8, seed=7, first=3, batch=7)
    for w, x, y in zip(whole, a, b):
        assert np.array_equal(w, np.concatenate([x, y]))
    other = oracle_mod.generate("sylvester", 8, seed=8, first=0, batch=1)
    assert not np.array_equal(other[2][0], whole[2][0])


def test_compulsory_bytes_model():
    # 12n^2+4n, 16n^2+8n, 24n^2+8n
    for n in (4, 64, 128):
        assert bytes_compulsory("cholesky", n) == 12 * n * n + 4 * n
        assert bytes_compulsory("lyapunov", n) == 16 * n * n + 8 * n
        assert bytes_compulsory("sylvester", n) == 24 * n * n + 8 * n


@pytest.mark.parametrize("eq", EQUATIONS)
def test_oracle_matches_reference_large_n(eq, oracle_mod):
    """n = 48 ... 128, every variant x default b, against the reference
    interpreter's projections (tests/golden/make_golden_large.py)."""
    import large_golden as lg
    d = lg.data(eq)
    vs = builtin_variants(eq)
    worst = 0.0
    cache = {}
    for (n, v, b), es in lg.groups(eq).items():
        if n not in cache:
            cache[n] = lg.inputs(oracle_mod, eq, n, d)
        X, info = oracle_mod.execute(eq, vs[v].statements, n, b, cache[n])
        assert (info == 0).all()
        worst = max(worst, lg.max_rel_err(X, d, es))
    assert worst <= 1e-13, worst


def test_serialised_reference_algorithms(oracle_mod):
    """The serialised live `Algorithm` objects (make_algorithm_fixtures.py):
    encode_algorithm gives exactly the frozen variant table's statement lists,
    the flop model gives the reference's dynamic counts, and the C oracle run
    from the encoded statements reproduces the reference interpreter's X."""
    from algorithm_fixtures import load
    from paper_1906_08613_b200.variants import (EQ_INPUTS, builtin_variants, encode_algorithm,
                                                 flop_count, stmts_key)
    cases, blocks = load()
    for name, (algs, inst, want) in cases.items():
        table = builtin_variants(name)
        assert [a.index for a in algs] == [v.index for v in table]
        ins = [np.ascontiguousarray(inst.bindings[nm], dtype=np.float64)[None] for nm in EQ_INPUTS[name]]
        for alg, v in zip(algs, table):
            stmts = encode_algorithm(alg)
            assert stmts_key(stmts) == stmts_key(v.statements)
            for b in blocks:
                x, flops = want[(alg.index, b)]
                assert flop_count(name, stmts, inst.n, b) == flops
                got, info = oracle_mod.execute(name, stmts, inst.n, b, ins)
                assert int(info[0]) == 0
                assert np.linalg.norm(got[0] - x) <= 1e-13 * max(1.0, np.linalg.norm(x))
