"""ctypes binding of the sm_100a kernel library (include/lagen_b200.h).

There is no CPU fallback: if the library is missing this module raises at
import time, and every solve goes through the CUDA entry points.
"""

import ctypes
from pathlib import Path

from . import errors

LIB_PATH = Path(__file__).resolve().parent / "lib" / "liblagen_b200.so"

LAGEN_OK = 0
STATUS_NAMES = {-1: "LAGEN_EINVAL", -2: "LAGEN_EUNSUPPORTED", -3: "LAGEN_EVARIANT", -4: "LAGEN_ECUDA"}


class View(ctypes.Structure):
    _fields_ = [("op", ctypes.c_int8), ("r", ctypes.c_int8),
                ("c", ctypes.c_int8), ("trans", ctypes.c_int8)]


class Stmt(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int8), ("sign", ctypes.c_int8),
                ("out", View), ("ins", View * 2)]


def _load():
    if not LIB_PATH.exists():
        raise ImportError(
            f"{LIB_PATH} is missing: build the sm_100a library first "
            "(python -m paper_1906_08613_b200.build); there is no CPU fallback")
    lib = ctypes.CDLL(str(LIB_PATH))
    vp, ll, i = ctypes.c_void_p, ctypes.c_longlong, ctypes.c_int
    lib.lagen_b200_abi_version.restype = i
    lib.lagen_b200_last_error.restype = ctypes.c_char_p
    lib.lagen_b200_num_variants.argtypes = [i]
    lib.lagen_b200_variant_stmts.argtypes = [i, i, vp, i]
    lib.lagen_b200_supported.argtypes = [i, i, i]
    lib.lagen_b200_geometry.argtypes = [i, i, i, vp, vp, vp, vp]
    lib.lagen_b200_execute.argtypes = [i, vp, i, i, i, ll, vp, vp, vp, vp]
    lib.lagen_b200_execute_engine.argtypes = [i, vp, i, i, i, ll, vp, vp, vp, vp, i]
    lib.lagen_b200_warp_supported.argtypes = [i, i, i, i]
    lib.lagen_b200_execute_profile.argtypes = [i, vp, i, i, i, ll, vp, vp, vp, vp, i, vp]
    lib.lagen_b200_engine_supported.argtypes = [i, i, i, i, i]
    lib.lagen_b200_execute_host.argtypes = [i, vp, i, i, i, ll, vp, vp, vp]
    lib.lagen_b200_execute_host_engine.argtypes = [i, vp, i, i, i, ll, vp, vp, vp, i]
    lib.lagen_b200_generate.argtypes = [i, i, ctypes.c_ulonglong, ll, ll, vp, vp]
    lib.lagen_b200_host_bytes.argtypes = [i, i, ll, vp, vp]
    lib.lagen_b200_execute_host_flags.argtypes = [i, vp, i, i, i, ll, vp, vp, vp, i, i]
    lib.lagen_b200_host_bytes_flags.argtypes = [i, i, ll, i, vp, vp]
    lib.lagen_b200_host_sync.argtypes = []
    lib.lagen_b200_cholesky.argtypes = [i, i, i, ll, vp, vp, vp, vp]
    lib.lagen_b200_lyapunov.argtypes = [i, i, i, ll, vp, vp, vp, vp, vp]
    lib.lagen_b200_sylvester.argtypes = [i, i, i, ll, vp, vp, vp, vp, vp, vp]
    return lib


lib = _load()
ABI_VERSION = lib.lagen_b200_abi_version()

EXPORTED = (
    "lagen_b200_abi_version", "lagen_b200_last_error", "lagen_b200_num_variants",
    "lagen_b200_variant_stmts", "lagen_b200_supported", "lagen_b200_geometry",
    "lagen_b200_cholesky", "lagen_b200_lyapunov", "lagen_b200_sylvester",
    "lagen_b200_execute", "lagen_b200_execute_host", "lagen_b200_execute_host_engine", "lagen_b200_generate",
    "lagen_b200_execute_engine", "lagen_b200_warp_supported", "lagen_b200_engine_supported",
    "lagen_b200_execute_profile", "lagen_b200_host_bytes", "lagen_b200_execute_host_flags",
    "lagen_b200_host_bytes_flags", "lagen_b200_host_sync",
)
HOST_TRIANGLES = 1
HOST_X_ZEROED = 2
HOST_ASYNC = 4
ENGINES = {"auto": 0, "generic": 1, "warp": 2, "column": 3, "dataflow": 4, "rows": 5, "wave": 6, "rowspad": 7, "pipe": 8, "rowsweep": 9, "rowsmix": 10}


def host_bytes(eq_code, n, batch, flags=0):
    """(H2D, D2H) bytes one host-pipeline call moves over PCIe."""
    h2d, d2h = ctypes.c_longlong(0), ctypes.c_longlong(0)
    check(lib.lagen_b200_host_bytes_flags(eq_code, n, batch, flags, ctypes.byref(h2d), ctypes.byref(d2h)),
          "host_bytes")
    return h2d.value, d2h.value


def engine_supported(eq_code, n, b, variant, engine):
    return bool(lib.lagen_b200_engine_supported(eq_code, n, b, variant, ENGINES[engine]))


def check(rc, what):
    """Map a negative status to the reference's error classes (errors.py)."""
    if rc == LAGEN_OK:
        return
    msg = lib.lagen_b200_last_error().decode(errors="replace")
    name = STATUS_NAMES.get(rc, str(rc))
    if rc == -2:
        raise errors.UnsupportedSizeError(f"{what}: {name}: {msg}")
    if rc == -3:
        raise errors.VariantError(f"{what}: {name}: {msg}")
    if rc == -4:
        raise errors.DeviceError(f"{what}: {name}: {msg}")
    raise errors.UsageError(f"{what}: {name}: {msg}")


def stmt_array(stmts):
    arr = (Stmt * len(stmts))()
    for k, s in enumerate(stmts):
        arr[k].kind = s["kind"]
        arr[k].sign = s["sign"]
        arr[k].out.op, arr[k].out.r, arr[k].out.c = s["out"][:3]
        arr[k].out.trans = 0
        for j in range(2):
            v = s["ins"][j]
            arr[k].ins[j].op, arr[k].ins[j].r, arr[k].ins[j].c, arr[k].ins[j].trans = v
    return arr


def geometry(eq_code, n, b):
    g, p, t, s = ctypes.c_int(), ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
    rc = lib.lagen_b200_geometry(eq_code, n, b, ctypes.byref(g), ctypes.byref(p),
                                 ctypes.byref(t), ctypes.byref(s))
    check(rc, "geometry")
    return {"threads_per_problem": g.value, "problems_per_cta": p.value,
            "threads_per_cta": t.value, "smem_bytes": s.value}
