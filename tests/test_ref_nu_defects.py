"""Regression fixtures for two defects of the REFERENCE's nu-mode CPU path
(SURVEY §0.4, §8f rank 4).  They guard the parity tooling: the CPU baseline
(oracle/_ref) must never contain a kernel hit by them.

1. Symmetric tile gather: `_nu_gemm` mirrors a symmetric diagonal operand
   with a doubly transposed tile index (ref:pkg/src/lagen/lowering.py:628-636,
   `tile_rc` at 623-626), so every nu-Lyapunov kernel whose GEMM reads a
   symmetric X view wider than one nu tile (b > nu) is wrong by O(1).
2. `.so` name collision: the emitted function name carries no mode
   (ref:pkg/src/lagen/lowering.py:952), so the reference's own equivalence
   test compiles the scalar and nu twins to one path and `ctypes.CDLL`
   returns the scalar library for both
   (ref:pkg/tests/test_acceptance.py:257-267) — the nu kernels never run there.

Runs where the reference tree and gcc are present (the build container);
the committed fixture tests/golden/nu_defect.json pins the observed numbers
so the finding is visible without the reference.
"""
import ctypes
import json
import os
import shutil
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

REPO = Path(__file__).resolve().parents[1]
REF = Path(os.environ.get("LAGEN_REFERENCE", "/root/reference"))
FIXTURE = REPO / "tests" / "golden" / "nu_defect.json"

needs_ref = pytest.mark.skipif(
    not (REF / "pkg" / "src" / "lagen").is_dir() or shutil.which("gcc") is None,
    reason="needs the reference tree and gcc (build container only)")


def _lagen():
    src = str(REF / "pkg" / "src")
    if src not in sys.path:
        sys.path.insert(0, src)
    import lagen  # noqa: F401
    return lagen


def _emit(eq_name, variant, n, b, mode):
    _lagen()
    from lagen.cli import VariantConfig, build_program
    from lagen.codegen import emit_function, emit_nu_kernel_header
    from lagen.lang import parse_equation
    from lagen.worksheet import enumerate_algorithms
    case = {"lyapunov": "lyapunov.la", "sylvester": "sylvester.la", "cholesky": "cholesky.la"}[eq_name]
    eq = parse_equation((REF / "pkg" / "cases" / case).read_text(), name=eq_name)
    alg = enumerate_algorithms(eq)[variant]
    cfg = VariantConfig(alg, variant, b, b, mode, 4 if mode == "nu" else None)
    return eq, alg, emit_function(build_program(cfg, n)), emit_nu_kernel_header(4)


def _compile_and_run(fn, header, so_path, inst, n):
    work = so_path.parent
    (work / "nu_kernels_4.h").write_text(header.text)
    src = work / (so_path.stem + ".c")
    src.write_text(fn.text)
    subprocess.run(["gcc", "-std=c99", "-O2", "-shared", "-fPIC", f"-I{work}", str(src), "-o", str(so_path), "-lm"],
                   check=True, capture_output=True)
    lib = ctypes.CDLL(str(so_path))
    bufs, args = [], []
    for pname, role in fn.params:
        m = np.ascontiguousarray(inst.bindings[pname]) if role == "in" else np.zeros((n, n))
        bufs.append((role, m))
        args.append(m.ctypes.data_as(ctypes.POINTER(ctypes.c_double)))
    getattr(lib, fn.name)(*args)
    return next(m for role, m in bufs if role == "out")


def _rel(got, want):
    return float(np.max(np.abs(got - want)) / max(1.0, float(np.max(np.abs(want)))))


@needs_ref
def test_nu_lyapunov_gather_defect_is_real_and_scalar_twin_is_fine(tmp_path):
    """nu-Lyapunov v5 at b = 8 (X11 spans 2x2 nu tiles) disagrees with the
    reference interpreter; its scalar twin and the b = 4 nu kernel agree."""
    from lagen.verify import interpret_algorithm, random_instance  # noqa: E402 (after _emit imports lagen)
    n = 16
    observed = {}
    for b, mode in ((8, "nu"), (8, "scalar"), (4, "nu")):
        eq, alg, fn, header = _emit("lyapunov", 5, n, b, mode)
        inst = random_instance(eq, n, seed=31)
        want, _ = interpret_algorithm(alg, inst, b)
        # per-mode .so name: the fix for the collision below
        got = _compile_and_run(fn, header, tmp_path / f"{fn.name}_{mode}.so", inst, n)
        observed[f"b{b}_{mode}"] = _rel(got, want["X"])
    assert observed["b8_nu"] > 1e-2, observed            # the defect: O(1) relative error
    assert observed["b8_scalar"] <= 1e-12, observed
    assert observed["b4_nu"] <= 1e-12, observed
    pinned = json.loads(FIXTURE.read_text())
    assert pinned["b8_nu_rel_err_min"] <= observed["b8_nu"]


@needs_ref
def test_scalar_and_nu_twins_share_one_function_and_so_name():
    """Same emitted symbol (and so the same `<name>.so` in the reference's
    test) for both modes: loading the second one by that path returns the
    first (ctypes caches dlopen handles by path)."""
    _, _, fs, _ = _emit("lyapunov", 5, 16, 8, "scalar")
    _, _, fnu, _ = _emit("lyapunov", 5, 16, 8, "nu")
    assert fs.name == fnu.name
    assert fs.text != fnu.text  # different code behind one name


@needs_ref
def test_collision_hides_the_defect(tmp_path):
    """Reproduce the reference test's flow: scalar then nu compiled to the
    SAME path while the first handle is alive -> the 'nu' call runs scalar
    code and the comparison passes vacuously."""
    from lagen.verify import interpret_algorithm, random_instance
    n, b = 16, 8
    eq, alg, fs, header = _emit("lyapunov", 5, n, b, "scalar")
    _, _, fnu, _ = _emit("lyapunov", 5, n, b, "nu")
    inst = random_instance(eq, n, seed=31)
    want, _ = interpret_algorithm(alg, inst, b)
    so = tmp_path / f"{fs.name}.so"
    x_scalar = _compile_and_run(fs, header, so, inst, n)
    keep = ctypes.CDLL(str(so))  # the reference's test keeps every handle alive
    x_nu_same_path = _compile_and_run(fnu, header, so, inst, n)
    assert keep is not None
    assert _rel(x_scalar, want["X"]) <= 1e-12
    assert _rel(x_nu_same_path, want["X"]) <= 1e-12      # vacuous: scalar code ran
    x_nu_own_path = _compile_and_run(fnu, header, tmp_path / f"{fnu.name}_nu.so", inst, n)
    assert _rel(x_nu_own_path, want["X"]) > 1e-2         # the same source, actually executed


def test_cpu_baseline_never_selects_an_affected_kernel():
    """oracle/build_ref.py: every candidate is checked against the reference
    interpreter, RefLib only offers verified kernels, and no nu-Lyapunov
    candidate has b > nu = 4."""
    from oracle import build_ref
    for v, b, mode in build_ref.CANDIDATES["lyapunov"]:
        assert not (mode == "nu" and b > 4), (v, b, mode)
    if not build_ref.available():
        pytest.skip("oracle/_ref not generated here")
    manifest = json.loads(build_ref.MANIFEST.read_text())["kernels"]
    assert manifest and all("verified" in k for k in manifest)
    for k in manifest:
        if k["verified"]:
            assert k["max_rel_err_vs_interpreter"] <= 1e-12
    ref = build_ref.RefLib.__new__(build_ref.RefLib)
    ref.manifest = manifest
    for eq in ("cholesky", "lyapunov", "sylvester"):
        for n in (16, 64, 128):
            offered = ref.kernels(eq, n)
            assert offered and all(k["verified"] for _, k in offered)


@needs_ref
def test_build_ref_verification_would_catch_the_defect(tmp_path, monkeypatch):
    """Feed the affected kernel through build_ref.generate's own check by
    adding it to the candidate list (scratch output directory)."""
    from oracle import build_ref
    monkeypatch.setattr(build_ref, "REF", tmp_path)
    monkeypatch.setattr(build_ref, "SRC", tmp_path / "src")
    monkeypatch.setattr(build_ref, "MANIFEST", tmp_path / "manifest.json")
    monkeypatch.setattr(build_ref, "SIZES", [16])
    monkeypatch.setattr(build_ref, "CANDIDATES", {"cholesky": [(1, 4, "nu")], "lyapunov": [(5, 8, "nu"), (5, 4, "nu")],
                                                  "sylvester": [(0, 4, "nu")]})
    kernels = build_ref.generate(REF)
    bad = [k for k in kernels if not k["verified"]]
    assert [(k["eq"], k["variant"], k["b"], k["mode"]) for k in bad] == [("lyapunov", 5, 8, "nu")]
    ref = build_ref.RefLib.__new__(build_ref.RefLib)
    ref.manifest = kernels
    assert all(k["b"] == 4 for _, k in ref.kernels("lyapunov", 16))


def test_fixture_records_the_finding():
    pinned = json.loads(FIXTURE.read_text())
    assert pinned["equation"] == "lyapunov" and pinned["b"] == 8 and pinned["mode"] == "nu"
    assert pinned["b8_nu_rel_err"] > 1e-2 and pinned["b8_scalar_rel_err"] <= 1e-12
