"""C-ABI boundary checks that need no GPU: the library loads, exports every
symbol include/lagen_b200.h declares, carries the reference's variant table,
and rejects malformed calls before touching the device."""

import ctypes
import re
from pathlib import Path

import pytest

from paper_1906_08613_b200 import _lib
from paper_1906_08613_b200.variants import EQ_CODES, EQUATIONS, builtin_variants, default_blocks

HEADER = Path(__file__).resolve().parents[1] / "include" / "lagen_b200.h"


def declared_symbols():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"\b(lagen_b200_\w+)\s*\(", text)))


def test_header_declares_what_python_binds():
    assert set(declared_symbols()) == set(_lib.EXPORTED)


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(str(_lib.LIB_PATH))
    for sym in declared_symbols():
        assert hasattr(lib, sym), sym


def test_abi_version():
    assert _lib.lib.lagen_b200_abi_version() == 1


@pytest.mark.parametrize("eq", EQUATIONS)
def test_variant_table_matches_reference_enumeration(eq):
    lib = _lib.lib
    vs = builtin_variants(eq)
    assert lib.lagen_b200_num_variants(EQ_CODES[eq]) == len(vs)
    for v in vs:
        arr = (_lib.Stmt * 16)()
        cnt = lib.lagen_b200_variant_stmts(EQ_CODES[eq], v.index, ctypes.addressof(arr), 16)
        assert cnt == len(v.statements)
        for k, s in enumerate(v.statements):
            got = arr[k]
            assert (got.kind, got.sign) == (s["kind"], s["sign"])
            assert (got.out.op, got.out.r, got.out.c) == tuple(s["out"])
            for j in range(2):
                gv = got.ins[j]
                assert (gv.op, gv.r, gv.c, gv.trans) == tuple(s["ins"][j])
    assert lib.lagen_b200_variant_stmts(EQ_CODES[eq], len(vs), None, 0) == -3


def test_every_size_and_default_block_is_instantiated():
    lib = _lib.lib
    for eq in range(3):
        for n in range(4, 129, 4):
            for b in default_blocks(n):
                assert lib.lagen_b200_supported(eq, n, b) == 1, (eq, n, b)
            assert lib.lagen_b200_supported(eq, n, 3) == 0
        assert lib.lagen_b200_supported(eq, 132, 4) == 0


def test_geometry_fits_the_sm():
    for eq in range(3):
        for n in range(4, 129, 4):
            for b in default_blocks(n):
                g = _lib.geometry(eq, n, b)
                assert g["threads_per_cta"] <= 1024
                assert g["smem_bytes"] <= 227 * 1024
                assert g["threads_per_cta"] == g["threads_per_problem"] * g["problems_per_cta"]


def _execute(eq, stmts, n, b, batch, inputs=None, X=None):
    arr = _lib.stmt_array(stmts) if stmts else None
    ptrs = inputs
    return _lib.lib.lagen_b200_execute(eq, ctypes.addressof(arr) if arr is not None else None,
                                       len(stmts) if stmts else 0, n, b, batch,
                                       ctypes.addressof(ptrs) if ptrs is not None else None, X, None, None)


def test_rejects_bad_arguments_without_a_device():
    v = builtin_variants("cholesky")[2].statements
    assert _execute(0, v, 16, 4, -1) == -1            # negative batch
    assert _execute(7, v, 16, 4, 1) == -1             # unknown equation
    assert _execute(0, v, 18, 4, 1) == -2             # b does not divide n
    assert _execute(0, v, 1028, 4, 1) == -2           # beyond LAGEN_BIG_MAX_N (132 now runs on the big engine)
    assert _execute(0, [], 16, 4, 1) == -3            # empty statement list
    bad = [dict(s) for s in v]
    bad[0] = dict(bad[0], kind=9)
    assert _execute(0, bad, 16, 4, 1) == -3           # unknown kind
    bad = [dict(s) for s in v]
    bad[2] = dict(bad[2], out=(1, 2, 2))
    assert _execute(0, bad, 16, 4, 1) == -3           # writes outside the output
    assert _execute(0, v, 16, 4, 1) == -1             # null buffers
    assert b"null" in _lib.lib.lagen_b200_last_error()
    assert _execute(0, v, 16, 4, 0) == 0              # empty batch is a no-op
    lyap = builtin_variants("lyapunov")[0].statements
    assert _execute(0, lyap, 16, 4, 1) == -3          # LYAP/SYLV inside Cholesky


def test_dispatch_table_points_at_instantiated_kernels():
    """Every autotuned (variant, b, engine) choice must exist in the library."""
    import json
    from paper_1906_08613_b200 import dispatch
    table = json.loads(dispatch.TABLE.read_text())
    assert set(table) == set(EQUATIONS)
    for eq, entries in table.items():
        assert len(entries) == 32, eq
        for n, e in entries.items():
            n = int(n)
            assert e["b"] in default_blocks(n) or e["b"] == n  # b = n: the leaf on the whole matrix
            assert 0 <= e["variant"] < len(builtin_variants(eq))
            assert _lib.engine_supported(EQ_CODES[eq], n, e["b"], e["variant"], e.get("engine", "generic")), (eq, n, e)


def test_every_variant_has_a_generic_kernel_at_every_size():
    """The generic engine covers the whole variant space (23 variants x default b x n)."""
    for eq in EQUATIONS:
        for n in range(4, 129, 4):
            for b in default_blocks(n):
                for v in builtin_variants(eq):
                    assert _lib.engine_supported(EQ_CODES[eq], n, b, v.index, "generic")


def test_emitted_kernel_builds_and_exports(tmp_path):
    """emit.py: a statement list -> one CUDA translation unit -> an sm_100a
    shared object exporting <eq>_v<k>_n<n>_b<b>_cuda with the reference's
    _signature order (codegen.py:143-152); no compute call without a GPU."""
    import ctypes
    from algorithm_fixtures import load
    from paper_1906_08613_b200 import emit
    cases, _ = load()
    algs, inst, _ = cases["sylvester"]
    mod = emit.emit_cuda("sylvester", algs[7], inst.n, 4)
    assert mod.name == "sylvester_v7_n16_b4_cuda"
    assert mod.text.count("    St<") == len(algs[7].statements)
    assert "const double* L, const double* U, const double* C, double* X" in mod.text
    so = emit.compile_module(mod, tmp_path)
    lib = ctypes.CDLL(str(so))
    assert hasattr(lib, mod.name)
    vals = [ctypes.c_int() for _ in range(4)]
    getattr(lib, mod.name + "_shape")(*[ctypes.byref(v) for v in vals])
    assert [v.value for v in vals] == [2, 16, 4, len(algs[7].statements)]
    with pytest.raises(Exception):
        emit.emit_cuda("sylvester", algs[7], 16, 5)


def test_big_engine_size_range():
    """128 < n <= LAGEN_BIG_MAX_N (b | n) is served by the big engine
    (bigsolve.cu) under engine auto / generic; nothing beyond it."""
    big = int(re.search(r"#define LAGEN_BIG_MAX_N (\d+)", HEADER.read_text()).group(1))
    assert big >= 256
    for eq in EQUATIONS:
        assert _lib.engine_supported(EQ_CODES[eq], 256, 16, 0, "generic")
        assert _lib.engine_supported(EQ_CODES[eq], big, 8, 0, "generic")
        assert not _lib.engine_supported(EQ_CODES[eq], big + 4, 4, 0, "generic")
        assert not _lib.engine_supported(EQ_CODES[eq], 256, 7, 0, "generic")
        assert not _lib.engine_supported(EQ_CODES[eq], 256, 8, 0, "warp")


def test_host_bytes_of_the_hybrid_triangle_transfer():
    """lagen_b200_host_bytes_flags counts what the host pipeline moves: with
    LAGEN_HOST_TRIANGLES and n >= 16 the copy engines take rows [0, s) of an
    upper part / rows [s, n) of a lower part at full width (s = n / 2 on the
    8-column grid) and the zero-copy kernels the remaining triangle."""
    from paper_1906_08613_b200 import executor
    n, batch = 64, 10
    s = 32
    upper = s * n + sum(n - 8 * (r // 8) for r in range(s, n))
    lower = (n - s) * n + sum(min(n, 8 * (r // 8) + 8) for r in range(s))
    assert upper == 2688 and lower == 2688
    h2d, d2h = _lib.host_bytes(EQ_CODES["cholesky"], n, batch, _lib.HOST_TRIANGLES | _lib.HOST_X_ZEROED)
    assert h2d == batch * upper * 8 and d2h == batch * (upper * 8 + 4)
    h2d, d2h = _lib.host_bytes(EQ_CODES["cholesky"], n, batch, _lib.HOST_TRIANGLES)
    assert h2d == batch * upper * 8 and d2h == batch * (n * n * 8 + 4)      # X comes back dense unless zeroed by the caller
    h2d, d2h = _lib.host_bytes(EQ_CODES["lyapunov"], n, batch, _lib.HOST_TRIANGLES)
    assert h2d == batch * (lower + upper) * 8 and d2h == batch * (n * n * 8 + 4)
    h2d, d2h = _lib.host_bytes(EQ_CODES["sylvester"], n, batch, _lib.HOST_TRIANGLES)
    assert h2d == batch * (lower + upper + n * n) * 8
    h2d, d2h = _lib.host_bytes(EQ_CODES["sylvester"], n, batch, 0)
    assert h2d == batch * 3 * n * n * 8 and d2h == batch * (n * n * 8 + 4)
    assert executor.host_triangles_default("cholesky", 16) and not executor.host_triangles_default("cholesky", 12)
    assert not executor.host_triangles_default("sylvester", 132)
