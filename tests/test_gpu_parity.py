"""GPU parity: the CUDA path (through the C ABI) against the reference.

  * golden vectors of the reference's interpret_algorithm, every variant,
    every default b and b = n, n in {4, 8, 12, 16, 24, 32}, two instance
    families; and projections of the reference's outputs at n in
    {48, 64, 96, 128}, every variant x default b (make_golden_large.py);
    every engine against the SAME (variant, b)'s reference output;
  * the CPU oracle (oracle/lagen_oracle.c, pinned to the reference by
    test_oracle_golden.py) on device-generated BASELINE inputs, every
    variant x b x engine at every n in 4..128 against the oracle's run of
    the same variant and b;
  * size-independent properties at full BASELINE batch sizes (residual,
    exact structure, shard invariance, host pipeline == device path).

Tolerances (BASELINE.json north_star): per-problem relative Frobenius
difference <= 1e-10 and residual ||op(X) - RHS||_F / ||RHS||_F <= 10 n eps.
"""

import json
from pathlib import Path

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from paper_1906_08613_b200 import errors, executor  # noqa: E402
from paper_1906_08613_b200.variants import (EQ_CODES, EQ_INPUTS, EQUATIONS,  # noqa: E402
                                             builtin_variants, default_blocks)

EPS = np.finfo(np.float64).eps
REL_TOL = 1e-10
GOLDEN = Path(__file__).resolve().parent / "golden"
META = json.loads((GOLDEN / "golden_meta.json").read_text())


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    torch.cuda.set_device(0)


# every engine of the C ABI (LAGEN_ENGINE_*), auto excluded
ENGINES = ("generic", "warp", "column", "dataflow", "rows", "wave", "rowspad", "pipe", "rowsweep", "rowsmix")


def blocks_of(n):
    """the reference's default blocks plus b = n (verify.py:232-233)"""
    return sorted(set(default_blocks(n)) | {n})


def engine_runs(eq, n, variants, blocks=None):
    from paper_1906_08613_b200 import _lib
    return [(v, b, e) for e in ENGINES for v in variants for b in (blocks or blocks_of(n))
            if _lib.engine_supported(EQ_CODES[eq], n, b, v, e)]


def rel_diff(X, Y):
    num = np.linalg.norm((X - Y).reshape(X.shape[0], -1), axis=1)
    den = np.maximum(1.0, np.linalg.norm(Y.reshape(Y.shape[0], -1), axis=1))
    return num / den


def to_dev(arrs):
    return [torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in arrs]


@pytest.mark.parametrize("eq", EQUATIONS)
def test_golden_reference_vectors(eq):
    d = np.load(GOLDEN / f"{eq}.npz")
    vs = builtin_variants(eq)
    worst = 0.0
    groups = {}
    for e in META[eq]["entries"]:
        groups.setdefault((e["n"], e["variant"], e["b"]), []).append(e)
    for (n, v, b), es in groups.items():
      for _, _, engine in engine_runs(eq, n, [v], [b]):
        ins = [np.stack([d[f"in_{e['case']}_{n}_{nm}"] for e in es]) for nm in EQ_INPUTS[eq]]
        X, info = executor.solve(eq, to_dev(ins), variant=v, b=b, engine=engine)
        X = X.cpu().numpy()
        want = np.stack([d[e["key"]] for e in es])
        assert (info.cpu().numpy() == 0).all()
        err = rel_diff(X, want).max()
        worst = max(worst, err)
        assert err <= REL_TOL, (eq, n, v, b, engine, err)
        if eq == "cholesky":
            assert np.all(np.tril(X, -1) == 0.0)
        if eq == "lyapunov":
            assert np.array_equal(X, np.transpose(X, (0, 2, 1)))
    print(f"{eq}: worst relative difference vs reference interpreter {worst:.3e}")


SWEEP_N = list(range(4, 129, 4))


@pytest.mark.parametrize("eq", EQUATIONS)
@pytest.mark.parametrize("n", SWEEP_N)
def test_every_variant_vs_oracle(eq, n, oracle_mod):
    batch = 48 if n <= 64 else 24
    ins_d = executor.generate(eq, n, seed=n, batch=batch)
    ins_h = [t.cpu().numpy() for t in ins_d]
    vs = builtin_variants(eq)
    res_tol = 10 * n * EPS
    refs = {}
    for v, b, engine in engine_runs(eq, n, [v.index for v in vs]):
        if (v, b) not in refs:  # the oracle's run of the same variant and block size
            ref_X, ref_info = oracle_mod.execute(eq, vs[v].statements, n, b, ins_h)
            assert (ref_info == 0).all()
            refs[(v, b)] = ref_X
        ref_X = refs[(v, b)]
        X, info = executor.solve(eq, ins_d, variant=v, b=b, engine=engine)
        X = X.cpu().numpy()
        assert (info.cpu().numpy() == 0).all(), (eq, n, v, b, engine)
        err = rel_diff(X, ref_X).max()
        assert err <= REL_TOL, (eq, n, v, b, engine, err)
        res = oracle_mod.residual(eq, n, ins_h, X)
        assert res.max() <= res_tol, (eq, n, v, b, engine, res.max() / (n * EPS))
        if eq == "cholesky":
            assert np.all(np.tril(X, -1) == 0.0)
        if eq == "lyapunov":
            assert np.array_equal(X, np.transpose(X, (0, 2, 1)))


@pytest.mark.parametrize("eq", EQUATIONS)
def test_large_n_reference_goldens(eq, oracle_mod):
    """n = 48, 64, 96, 128: every engine x variant x default b against the
    reference interpreter's own output for the same (variant, b), through
    its projections (tests/golden/make_golden_large.py)."""
    import large_golden as lg
    d = lg.data(eq)
    cache = {}
    worst = 0.0
    for (n, v, b), es in lg.groups(eq).items():
        if n not in cache:
            cache[n] = to_dev(lg.inputs(oracle_mod, eq, n, d))
        for _, _, engine in engine_runs(eq, n, [v], [b]):
            X, info = executor.solve(eq, cache[n], variant=v, b=b, engine=engine)
            assert (info.cpu().numpy() == 0).all(), (eq, n, v, b, engine)
            err = lg.max_rel_err(X.cpu().numpy(), d, es)
            worst = max(worst, err)
            assert err <= REL_TOL, (eq, n, v, b, engine, err)
    print(f"{eq}: worst projected relative difference vs reference at n >= 48: {worst:.3e}")


@pytest.mark.parametrize("eq", EQUATIONS)
@pytest.mark.parametrize("n", [12, 16, 64, 124])
def test_every_engine_multi_round(eq, n, oracle_mod):
    """Batches larger than one round of resident problem slots, with a
    partial last round: every engine's loop-carried path (persistent CTAs,
    prefetch, slot reuse) against the oracle on the first and last problems."""
    batch = {12: 40001, 16: 30001, 64: 4001, 124: 1201}[n]
    ins_d = executor.generate(eq, n, seed=5 * n, batch=batch)
    pick = np.r_[0:16, batch - 16:batch]
    sub = [t[pick].cpu().numpy() for t in ins_d]
    vs = builtin_variants(eq)
    seen = set()
    for v, b, engine in engine_runs(eq, n, [v.index for v in vs]):
        if (engine, b) in seen:  # one variant per engine and block size keeps this test short
            continue
        seen.add((engine, b))
        X, info = executor.solve(eq, ins_d, variant=v, b=b, engine=engine)
        assert int((info != 0).sum()) == 0, (eq, n, v, b, engine)
        ref, _ = oracle_mod.execute(eq, vs[v].statements, n, b, sub)
        err = rel_diff(X[torch.from_numpy(pick).cuda()].cpu().numpy(), ref).max()
        assert err <= REL_TOL, (eq, n, v, b, engine, err)


ODD_N = [1, 2, 3, 5, 6, 7, 9, 10, 13, 18, 30, 31, 33, 47, 63, 66, 97, 127]


@pytest.mark.parametrize("eq", EQUATIONS)
@pytest.mark.parametrize("n", ODD_N)
def test_sizes_without_instance_vs_oracle(eq, n, oracle_mod):
    """n not a multiple of 4 (BASELINE target: every n in 4..128): the
    identity-padded path of the C ABI against the oracle's own (n, b) run,
    for every variant, with the reference's admissible b (b | n)."""
    batch = 32
    ins_d = executor.generate(eq, n, seed=1000 + n, batch=batch)
    ins_h = [t.cpu().numpy() for t in ins_d]
    blocks = sorted({b for b in (1, 2, 4, 8, n) if n % b == 0})
    res_tol = 10 * max(n, 4) * EPS
    for v in builtin_variants(eq):
        for b in blocks:
            ref_X, ref_info = oracle_mod.execute(eq, v.statements, n, b, ins_h)
            assert (ref_info == 0).all()
            X, info = executor.solve(eq, ins_d, variant=v.index, b=b)
            X = X.cpu().numpy()
            assert X.shape == (batch, n, n)
            assert (info.cpu().numpy() == 0).all(), (eq, n, v.index, b)
            err = rel_diff(X, ref_X).max()
            assert err <= REL_TOL, (eq, n, v.index, b, err)
            res = oracle_mod.residual(eq, n, ins_h, X)
            assert res.max() <= res_tol, (eq, n, v.index, b, res.max() / (n * EPS))
    # default selection (dispatch fallback b) and the host pipeline agree
    X0, _ = executor.solve(eq, ins_d)
    Xh, _ = executor.solve_host(eq, ins_h)
    assert np.array_equal(np.asarray(Xh), X0.cpu().numpy())


def test_padded_sizes_report_non_spd_index():
    n = 7
    A = torch.eye(n, dtype=torch.float64, device="cuda").repeat(2, 1, 1)
    A[1, 5, 5] = -1.0
    with pytest.raises(errors.VerificationError, match="index 5"):
        executor.solve("cholesky", [A], variant=1, b=1)
    _, info = executor.solve("cholesky", [A], variant=1, b=7, check=False)
    assert info.cpu().tolist() == [0, 6]
    with pytest.raises(errors.LagenError):
        executor.solve("cholesky", [A], variant=1, b=2)  # 2 does not divide 7 (verify.py:232-233)


def test_known_answers():
    for n in (4, 8, 16, 64):
        I = torch.eye(n, dtype=torch.float64, device="cuda").expand(3, n, n).contiguous()
        for v in builtin_variants("cholesky"):
            for b in default_blocks(n):
                X, _ = executor.solve("cholesky", [I], variant=v.index, b=b)
                assert torch.equal(X, I)
    n = 8
    L = (2.0 * torch.eye(n, dtype=torch.float64, device="cuda")).expand(2, n, n).contiguous()
    U = (3.0 * torch.eye(n, dtype=torch.float64, device="cuda")).expand(2, n, n).contiguous()
    C = torch.full((2, n, n), 10.0, dtype=torch.float64, device="cuda")
    for v in builtin_variants("sylvester"):
        X, _ = executor.solve("sylvester", [L, U, C], variant=v.index, b=4)
        assert torch.equal(X, torch.full_like(C, 2.0))


def test_non_spd_and_nan_are_reported():
    """info = first non-positive pivot + 1 (kernels.py:87-88) / -1 for NaN-Inf,
    on every engine that has the variant."""
    from paper_1906_08613_b200 import _lib
    for n, bad in ((16, 6), (32, 20), (44, 30), (48, 37)):
        A = executor.generate("cholesky", n, seed=1, batch=4)[0]
        A[2, bad, bad] = -1000.0
        with pytest.raises(errors.VerificationError):
            executor.solve("cholesky", [A], variant=2, b=4)
        for v in (1, 2):
            for engine in ("generic", "warp", "column", "dataflow", "rows", "rowspad", "rowsmix"):
                if not _lib.engine_supported(0, n, 4, v, engine):
                    continue
                X, info = executor.solve("cholesky", [A], variant=v, b=4, check=False, engine=engine)
                assert info.cpu().tolist() == [0, 0, bad + 1, 0], (n, v, engine)
        L, U, C = executor.generate("sylvester", n, seed=1, batch=3)
        C[1, 0, 0] = float("nan")
        for engine in ENGINES:
            for b in (4, n):
                if not _lib.engine_supported(2, n, b, 13, engine):
                    continue
                _, info = executor.solve("sylvester", [L, U, C], variant=13, b=b, check=False, engine=engine)
                assert info.cpu().tolist() == [0, -1, 0], (n, b, engine)
        L, S = executor.generate("lyapunov", n, seed=1, batch=3)
        S[2, n - 1, n - 1] = float("inf")
        for engine in ENGINES:
            for b in (4, n):
                if not _lib.engine_supported(1, n, b, 5, engine):
                    continue
                _, info = executor.solve("lyapunov", [L, S], variant=5, b=b, check=False, engine=engine)
                assert info.cpu().tolist() == [0, 0, -1], (n, b, engine)
    try:
        import lagen.errors
        with pytest.raises(lagen.errors.VerificationError):
            executor.solve("sylvester", [L, U, C], variant=13, b=4)
    except ImportError:
        pass


@pytest.mark.parametrize("eq", EQUATIONS)
def test_generator_matches_cpu_twin(eq, oracle_mod):
    for n in (4, 36, 128):
        dev = [t.cpu().numpy() for t in executor.generate(eq, n, seed=11, batch=5, first=1000)]
        cpu = oracle_mod.generate(eq, n, seed=11, first=1000, batch=5)
        for a, b in zip(dev, cpu):
            assert np.array_equal(a == 0.0, b == 0.0)
            np.testing.assert_allclose(a, b, rtol=1e-12, atol=1e-13)


@pytest.mark.parametrize("eq", EQUATIONS)
def test_shard_invariance_on_device(eq):
    n = 24
    whole = executor.generate(eq, n, seed=7, batch=40)
    lo = executor.generate(eq, n, seed=7, batch=17)
    hi = executor.generate(eq, n, seed=7, batch=23, first=17)
    for w, a, b in zip(whole, lo, hi):
        assert torch.equal(w, torch.cat([a, b]))
    Xw, _ = executor.solve(eq, whole)
    Xa, _ = executor.solve(eq, lo)
    Xb, _ = executor.solve(eq, hi)
    assert torch.equal(Xw, torch.cat([Xa, Xb]))


@pytest.mark.parametrize("eq", EQUATIONS)
def test_host_pipeline_equals_device_path(eq):
    n = 32
    ins = executor.generate(eq, n, seed=3, batch=70000 if eq == "cholesky" else 9000)
    Xd, _ = executor.solve(eq, ins)
    host = [t.cpu().pin_memory() for t in ins]
    Xh, info = executor.solve_host(eq, host)
    assert torch.equal(Xh, Xd.cpu())
    assert int(info.abs().sum()) == 0


def _device_residual(eq, ins, X):
    if eq == "cholesky":
        (A,) = ins
        R = torch.bmm(X.transpose(1, 2), X) - A
        rhs = A
    elif eq == "lyapunov":
        L, S = ins
        R = torch.bmm(L, X) + torch.bmm(X, L.transpose(1, 2)) - S
        rhs = S
    else:
        L, U, C = ins
        R = torch.bmm(L, X) + torch.bmm(X, U) - C
        rhs = C
    num = torch.linalg.matrix_norm(R)
    den = torch.clamp(torch.linalg.matrix_norm(rhs), min=1.0)
    return (num / den).cpu().numpy()


@pytest.mark.parametrize("eq", EQUATIONS)
@pytest.mark.parametrize("n", [16, 64, 128])
def test_full_batch_properties(eq, n, oracle_mod):
    """BASELINE batch floor(2^28 / 8n^2) (config 2-4 size): residual of every
    problem, plus a sampled oracle comparison."""
    batch = (1 << 28) // (8 * n * n)
    ins = executor.generate(eq, n, seed=n, batch=batch)
    X, info = executor.solve(eq, ins)
    assert int((info != 0).sum()) == 0
    res = _device_residual(eq, ins, X)
    assert res.max() <= 10 * n * EPS, res.max() / (n * EPS)
    idx = torch.randperm(batch, generator=torch.Generator().manual_seed(n))[:64].cuda()
    sub = [t[idx].cpu().numpy() for t in ins]
    vs = builtin_variants(eq)
    ref, _ = oracle_mod.execute(eq, vs[0].statements, n, default_blocks(n)[0], sub)
    assert rel_diff(X[idx].cpu().numpy(), ref).max() <= REL_TOL


def test_reference_algorithm_objects_drop_in():
    """The reference's own Algorithm objects run unchanged through the backend."""
    lagen = pytest.importorskip("lagen")
    from lagen.lang import parse_equation
    from lagen.verify import interpret_algorithm as ref_interpret, random_instance
    from lagen.worksheet import enumerate_algorithms

    cases = {
        "cholesky": "Equation: X^T * X = A\nA: Matrix(n,n), spd, input\nX: Matrix(n,n), upper_triangular, output\n",
        "lyapunov": "Equation: L * X + X * L^T = S\nL: Matrix(n,n), lower_triangular, input\n"
                    "S: Matrix(n,n), symmetric, input\nX: Matrix(n,n), symmetric, output\n",
        "sylvester": "Equation: L * X + X * U = C\nL: Matrix(n,n), lower_triangular, input\n"
                     "U: Matrix(n,n), upper_triangular, input\nC: Matrix(n,n), general, input\n"
                     "X: Matrix(n,n), general, output\n",
    }
    for name, text in cases.items():
        eq = parse_equation(text, name=name)
        inst = random_instance(eq, 16, seed=42)
        for alg in enumerate_algorithms(eq):
            for b in (4, 8):
                want, wflops = ref_interpret(alg, inst, b)
                got, gflops = executor.interpret_algorithm(alg, inst, b)
                assert gflops == wflops
                x = want["X"]
                assert np.linalg.norm(got["X"] - x) <= REL_TOL * max(1.0, np.linalg.norm(x))


def test_reference_algorithm_fixtures_drop_in():
    """The same drop-in on objects rebuilt from the serialised live
    `Algorithm`s (tests/golden/make_algorithm_fixtures.py): runs where the
    reference package is absent; expected X and flops are the reference
    interpreter's own (verify.py:221-303)."""
    from algorithm_fixtures import load
    cases, blocks = load()
    for name, (algs, inst, want) in cases.items():
        assert len(algs) == len(builtin_variants(name))
        for alg in algs:
            for b in blocks:
                x, wflops = want[(alg.index, b)]
                got, gflops = executor.interpret_algorithm(alg, inst, b)
                assert gflops == wflops
                assert np.linalg.norm(got[alg.output] - x) <= REL_TOL * max(1.0, np.linalg.norm(x))


def test_emitted_kernels_from_algorithm_objects():
    """f2: every synthesised variant emitted as its own compiled sm_100a kernel
    (emit.py, the counterpart of codegen.emit_function) from the serialised
    live `Algorithm` objects, against the reference interpreter's X for the
    same variant and b; and through executor.solve(engine="emitted")."""
    from concurrent.futures import ThreadPoolExecutor
    from algorithm_fixtures import load
    from paper_1906_08613_b200 import emit
    cases, blocks = load()
    jobs = [(name, alg, inst, b, want[(alg.index, b)][0])
            for name, (algs, inst, want) in cases.items() for alg in algs for b in blocks]
    with ThreadPoolExecutor(8) as ex:
        kernels = list(ex.map(lambda j: emit.compile_variant(j[0], j[1], j[2].n, j[3]), jobs))
    for (name, alg, inst, b, x), k in zip(jobs, kernels):
        assert k.name == f"{name}_v{alg.index}_n{inst.n}_b{b}_cuda"
        ins = [torch.from_numpy(np.ascontiguousarray(inst.bindings[nm], dtype=np.float64))[None].cuda()
               for nm in EQ_INPUTS[name]]
        X, info = k.solve(ins)
        assert int(info[0]) == 0
        assert np.linalg.norm(X[0].cpu().numpy() - x) <= REL_TOL * max(1.0, np.linalg.norm(x)), (name, alg.index, b)
        X2, _ = executor.solve(name, ins, variant=alg, b=b, engine="emitted")
        assert torch.equal(X2, X)
    # a batch with a partial last round, at a size beyond the fixtures, against the generic engine
    for name, v, n, b in (("sylvester", 7, 40, 8), ("lyapunov", 2, 36, 4), ("cholesky", 0, 64, 16)):
        ins = executor.generate(name, n, seed=n, batch=1000)
        X, _ = executor.solve(name, ins, variant=v, b=b, engine="emitted")
        R, _ = executor.solve(name, ins, variant=v, b=b, engine="generic")
        assert rel_diff(X.cpu().numpy(), R.cpu().numpy()).max() <= REL_TOL


@pytest.mark.parametrize("eq", EQUATIONS)
def test_sizes_beyond_128(eq, oracle_mod):
    """f3: 128 < n <= LAGEN_BIG_MAX_N on the big engine (bigsolve.cu) — the
    reference interpreter has no size limit (verify.py:221-303): every variant
    x b in {4, 8, 16} at n = 144, the dispatch default at n = 132, 192, 256,
    b = n, and the host path, against the oracle's run of the same (variant, b);
    a non-SPD / NaN input is reported like at the small sizes."""
    vs = builtin_variants(eq)
    cases = [(144, v.index, b, 5) for v in vs for b in (4, 8, 16)]
    cases += [(132, len(vs) - 1, 4, 3), (192, 1, 8, 700), (256, len(vs) - 1, 16, 3), (160, 0, 160, 2)]
    for n, v, b, batch in cases:
        host = oracle_mod.generate(eq, n, seed=n, first=0, batch=min(batch, 8))
        if batch > 8:  # more problems than resident CTAs: the grid-stride loop
            host = [np.concatenate([a] * (batch // 8 + 1))[:batch] for a in host]
        ins = [torch.from_numpy(a).cuda() for a in host]
        X, info = executor.solve(eq, ins, variant=v, b=b, check=False)
        assert int((info != 0).sum()) == 0
        k = min(batch, 8)
        ref, rinfo = oracle_mod.execute(eq, vs[v].statements, n, b, [a[:k] for a in host])
        assert (rinfo == 0).all()
        got = X.cpu().numpy()
        assert rel_diff(got[:k], ref).max() <= REL_TOL, (n, v, b)
        if batch > 8:
            assert np.array_equal(got, got[np.arange(batch) % 8])  # every round of the loop, same bits
        res = oracle_mod.residual(eq, n, [a[:k] for a in host], got[:k])
        assert res.max() <= 10 * n * EPS, (n, v, b, res.max() / (n * EPS))
    n = 136
    host = oracle_mod.generate(eq, n, seed=1, first=0, batch=3)
    Xh, ih = executor.solve_host(eq, host, variant=0, b=8)
    ref, _ = oracle_mod.execute(eq, vs[0].statements, n, 8, host)
    assert rel_diff(np.asarray(Xh), ref).max() <= REL_TOL and int(np.abs(np.asarray(ih)).sum()) == 0
    ins = [torch.from_numpy(a).cuda() for a in host]
    if eq == "cholesky":
        ins[0][1, 130, 130] = -1e6
        want = [0, 131, 0]
    else:
        ins[-1][1, 3, 5] = float("nan")
        want = [0, -1, 0]
    _, info = executor.solve(eq, ins, variant=len(vs) - 1, b=8, check=False)
    assert info.cpu().tolist() == want
    with pytest.raises(errors.UnsupportedSizeError):
        executor.solve(eq, [torch.zeros(1, 1028, 1028, dtype=torch.float64, device="cuda")] * len(ins), variant=0, b=4)


def test_host_pipeline_async_sequence():
    """solve_host(..., wait=False): several batches of different sizes and
    equations queued back to back on the same pipeline streams, one
    host_sync(); every result equals the device path bit for bit."""
    jobs = []
    for eq, n, batch in (("cholesky", 64, 3000), ("sylvester", 24, 5000), ("lyapunov", 96, 900),
                         ("cholesky", 12, 20000), ("cholesky", 100, 700)):
        ins = executor.generate(eq, n, seed=n, batch=batch)
        want, _ = executor.solve(eq, ins)
        host = [t.cpu().pin_memory() for t in ins]
        out = torch.zeros((batch, n, n), dtype=torch.float64).pin_memory()
        info = torch.full((batch,), 7, dtype=torch.int32).pin_memory()
        executor.solve_host(eq, host, out=out, info=info, out_zeroed=eq == "cholesky", wait=False)
        jobs.append((want.cpu(), out, info))
    executor.host_sync()
    for want, out, info in jobs:
        assert torch.equal(out, want)
        assert int(info.abs().sum()) == 0
    executor.host_sync()  # idempotent


@pytest.mark.parametrize("eq", EQUATIONS)
def test_config5_sampled(eq, oracle_mod):
    """BASELINE config 5 on one GPU: n = 64, 2^20 problems (2^32 doubles per
    operand, past the 2^31-element line), seed 7; every problem's info, the
    last 64 problems (largest offsets) and 64 spread ones against the oracle."""
    n, batch = 64, 1 << 20
    ins = executor.generate(eq, n, seed=7, batch=batch)
    X, info = executor.solve(eq, ins, check=False)
    assert int((info != 0).sum()) == 0
    pick = np.r_[np.linspace(0, batch - 65, 64).astype(np.int64), batch - 64:batch]
    idx = torch.from_numpy(pick).cuda()
    sub = [t[idx].cpu().numpy() for t in ins]
    from paper_1906_08613_b200 import dispatch
    sel = dispatch.select(eq, n)
    ref, rinfo = oracle_mod.execute(eq, builtin_variants(eq)[sel["variant"]].statements, n,
                                    sel["b"] if n % sel["b"] == 0 else default_blocks(n)[0], sub)
    assert (rinfo == 0).all()
    assert rel_diff(X[idx].cpu().numpy(), ref).max() <= REL_TOL
    # the generator is index-keyed: the last problems equal a fresh generation at their offset
    tail = executor.generate(eq, n, seed=7, batch=64, first=batch - 64)
    for a, b in zip(ins, tail):
        assert torch.equal(a[batch - 64:], b)
    del ins, X
    torch.cuda.empty_cache()


def test_typed_entry_points_against_goldens():
    """lagen_b200_cholesky / _lyapunov / _sylvester — the replacements of the
    emitted kernel <eq>_v<k>_n<n>_b<b>(inputs..., X) (codegen.py:143-201) —
    called through ctypes on the reference's golden inputs."""
    import ctypes
    from paper_1906_08613_b200 import _lib
    fns = {"cholesky": _lib.lib.lagen_b200_cholesky, "lyapunov": _lib.lib.lagen_b200_lyapunov,
           "sylvester": _lib.lib.lagen_b200_sylvester}
    for eq in EQUATIONS:
        d = np.load(GOLDEN / f"{eq}.npz")
        for e in META[eq]["entries"]:
            if e["case"] != "base" or e["n"] not in (8, 24, 32):
                continue
            n = e["n"]
            ins = to_dev([d[f"in_base_{n}_{nm}"][None] for nm in EQ_INPUTS[eq]])
            X = torch.full((1, n, n), float("nan"), dtype=torch.float64, device="cuda")  # every entry is written
            info = torch.full((1,), 7, dtype=torch.int32, device="cuda")
            ptrs = [ctypes.c_void_p(t.data_ptr()) for t in ins]
            rc = fns[eq](e["variant"], n, e["b"], 1, *ptrs, ctypes.c_void_p(X.data_ptr()),
                         ctypes.c_void_p(info.data_ptr()), ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
            assert rc == 0, _lib.lib.lagen_b200_last_error()
            torch.cuda.synchronize()
            assert int(info[0]) == 0
            want = d[e["key"]][None]
            assert rel_diff(X.cpu().numpy(), want).max() <= REL_TOL, (eq, e["key"])
    # errors come back as status codes, not exceptions
    A = torch.zeros((1, 8, 8), dtype=torch.float64, device="cuda")
    assert _lib.lib.lagen_b200_cholesky(0, 8, 3, 1, ctypes.c_void_p(A.data_ptr()), ctypes.c_void_p(A.data_ptr()),
                                        None, None) == -2
    assert _lib.lib.lagen_b200_cholesky(99, 8, 4, 1, ctypes.c_void_p(A.data_ptr()), ctypes.c_void_p(A.data_ptr()),
                                        None, None) == -3


@pytest.mark.parametrize("eq", ["lyapunov", "sylvester"])
def test_padded_sizes_with_minus_one_diagonal(eq, oracle_mod):
    """n not a multiple of 4 runs identity-padded in the C ABI; a real
    diagonal entry of -1 must not meet a padded pivot of +1 (0 / 0): the pad
    value is 1 + max |diagonal| per problem."""
    for n in (6, 30):
        ins = executor.generate(eq, n, seed=3, batch=4)
        # well-conditioned pivots around the -1 entries: the other diagonal
        # entries of those problems are 3 (pivots -1 + 3, 3 + 3, -1 - 1)
        for p, (op, k) in ((1, (0, 2)), (2, (1 if eq == "sylvester" else 0, n - 1))):
            for t in ins[:-1]:
                t[p].diagonal().fill_(3.0)
            ins[op][p, k, k] = -1.0
        ins_h = [t.cpu().numpy() for t in ins]
        for v in (0, len(builtin_variants(eq)) - 1):
            for b in sorted({1, 2, n} & {d for d in range(1, n + 1) if n % d == 0}):
                X, info = executor.solve(eq, ins, variant=v, b=b, check=False)
                assert info.cpu().tolist() == [0, 0, 0, 0], (eq, n, v, b)
                ref, _ = oracle_mod.execute(eq, builtin_variants(eq)[v].statements, n, b, ins_h)
                assert rel_diff(X.cpu().numpy(), ref).max() <= REL_TOL


@pytest.mark.parametrize("eq", EQUATIONS)
def test_unread_triangles_are_ignored(eq):
    """The structurally unused triangles (A's and S's strict lower, L's strict
    upper, U's strict lower — never read by the reference either,
    test_acceptance.py:167-184) may hold anything: NaN there changes nothing,
    on every engine x variant x b.  This is what lets the host path move
    triangles only."""
    for n in (16, 64):
        ins = executor.generate(eq, n, seed=9, batch=8)
        dirty = [t.clone() for t in ins]
        lower = torch.tril(torch.ones(n, n, dtype=torch.bool, device="cuda"), -1)
        if eq == "cholesky":
            dirty[0][:, lower] = float("nan")
        elif eq == "lyapunov":
            dirty[0][:, lower.T] = float("nan")
            dirty[1][:, lower] = float("nan")
        else:
            dirty[0][:, lower.T] = float("nan")
            dirty[1][:, lower] = float("nan")
        for v, b, engine in engine_runs(eq, n, [v.index for v in builtin_variants(eq)]):
            X0, _ = executor.solve(eq, ins, variant=v, b=b, engine=engine)
            X1, info = executor.solve(eq, dirty, variant=v, b=b, engine=engine, check=False)
            assert int(info.abs().sum()) == 0, (eq, n, v, b, engine)
            assert torch.equal(X0, X1), (eq, n, v, b, engine)


@pytest.mark.parametrize("eq", EQUATIONS)
def test_host_triangles_equal_device_path(eq):
    """solve_host moving triangles only (zero-copy from pinned memory), with
    and without the caller-zeroed X of the reference contract, equals the
    device path bit for bit; unpinned buffers and odd n take the dense path."""
    from paper_1906_08613_b200 import _lib
    for n in (16, 62, 128):
        batch = 3000 if n < 100 else 700
        ins = executor.generate(eq, n, seed=4, batch=batch)
        Xd, _ = executor.solve(eq, ins)
        host = [t.cpu().pin_memory() for t in ins]
        for zeroed in ((False, True) if eq == "cholesky" else (False,)):
            out = torch.zeros((batch, n, n), dtype=torch.float64).pin_memory() if zeroed else \
                torch.full((batch, n, n), float("nan"), dtype=torch.float64).pin_memory()
            Xh, info = executor.solve_host(eq, host, out=out, triangles=True, out_zeroed=zeroed)
            assert int(info.abs().sum()) == 0
            assert torch.equal(Xh, Xd.cpu()), (eq, n, zeroed)
        h2d, d2h = _lib.host_bytes(EQ_CODES[eq], n, batch, _lib.HOST_TRIANGLES)
        assert h2d < len(ins) * batch * n * n * 8
    with pytest.raises(errors.LagenError):
        executor.solve_host(eq, [t.cpu() for t in executor.generate(eq, 16, seed=4, batch=4)], triangles=True)
