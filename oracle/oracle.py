"""ctypes wrapper of the CPU oracle (lagen_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's CPU-baseline legs as the checker / reported baseline.  The product
package never imports this module.
"""

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "liblagen_oracle.so"

EQ_CODES = {"cholesky": 0, "lyapunov": 1, "sylvester": 2}
EQ_NINPUTS = {"cholesky": 1, "lyapunov": 2, "sylvester": 3}


class _View(ctypes.Structure):
    _fields_ = [("op", ctypes.c_int8), ("r", ctypes.c_int8),
                ("c", ctypes.c_int8), ("trans", ctypes.c_int8)]


class _Stmt(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int8), ("sign", ctypes.c_int8),
                ("out", _View), ("ins", _View * 2)]


def build(force=False):
    if LIB_PATH.exists() and not force:
        src = HERE / "lagen_oracle.c"
        if LIB_PATH.stat().st_mtime >= src.stat().st_mtime:
            return LIB_PATH
    subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
    return LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        _lib = ctypes.CDLL(str(LIB_PATH))
        dp = ctypes.POINTER(ctypes.c_double)
        _lib.oracle_execute.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_int,
                                        ctypes.c_int, ctypes.c_int, ctypes.c_longlong,
                                        ctypes.c_void_p, dp, ctypes.c_void_p, ctypes.c_int]
        _lib.oracle_residual.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_longlong,
                                         ctypes.c_void_p, dp, dp, ctypes.c_int]
        _lib.oracle_generate.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_ulonglong,
                                         ctypes.c_longlong, ctypes.c_longlong,
                                         ctypes.c_void_p, ctypes.c_int]
        _lib.oracle_chol_textbook.argtypes = [ctypes.c_int, ctypes.c_longlong, dp, dp,
                                              ctypes.c_void_p]
    return _lib


def stmt_array(stmts):
    arr = (_Stmt * len(stmts))()
    for i, s in enumerate(stmts):
        arr[i].kind = s["kind"]
        arr[i].sign = s["sign"]
        arr[i].out.op, arr[i].out.r, arr[i].out.c = s["out"][:3]
        arr[i].out.trans = 0
        for j in range(2):
            v = s["ins"][j]
            arr[i].ins[j].op, arr[i].ins[j].r, arr[i].ins[j].c, arr[i].ins[j].trans = v
    return arr


def _dptr(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _ptr_array(arrs):
    return (ctypes.c_void_p * len(arrs))(*[a.ctypes.data for a in arrs])


def _threads(nthreads):
    if nthreads is None:
        return len(os.sched_getaffinity(0))
    return nthreads


def execute(eq, stmts, n, b, inputs, nthreads=None):
    """Batched restatement of interpret_algorithm; inputs: arrays [batch, n, n].

    Returns (X, info)."""
    inputs = [np.ascontiguousarray(a, dtype=np.float64) for a in inputs]
    batch = inputs[0].shape[0]
    X = np.empty((batch, n, n))
    info = np.zeros(batch, dtype=np.int32)
    arr = stmt_array(stmts)
    ptrs = _ptr_array(inputs)
    rc = lib().oracle_execute(EQ_CODES[eq], ctypes.addressof(arr), len(stmts), n, b, batch,
                              ctypes.addressof(ptrs), _dptr(X),
                              info.ctypes.data, _threads(nthreads))
    if rc != 0:
        raise ValueError(f"oracle_execute failed with {rc}")
    return X, info


def residual(eq, n, inputs, X, nthreads=None):
    inputs = [np.ascontiguousarray(a, dtype=np.float64) for a in inputs]
    X = np.ascontiguousarray(X, dtype=np.float64)
    batch = X.shape[0]
    res = np.empty(batch)
    ptrs = _ptr_array(inputs)
    lib().oracle_residual(EQ_CODES[eq], n, batch, ctypes.addressof(ptrs),
                          _dptr(X), _dptr(res), _threads(nthreads))
    return res


def generate(eq, n, seed, first, batch, nthreads=None):
    outs = [np.empty((batch, n, n)) for _ in range(EQ_NINPUTS[eq])]
    ptrs = _ptr_array(outs)
    lib().oracle_generate(EQ_CODES[eq], n, seed, first, batch,
                          ctypes.addressof(ptrs), _threads(nthreads))
    return outs


def chol_textbook(A):
    A = np.ascontiguousarray(A, dtype=np.float64)
    batch, n, _ = A.shape
    X = np.empty_like(A)
    info = np.zeros(batch, dtype=np.int32)
    lib().oracle_chol_textbook(n, batch, _dptr(A), _dptr(X), info.ctypes.data)
    return X, info


def kron_solve(l, u, c):
    """verify.py:123-131 restated: (I (x) L + U^T (x) I) vec X = vec C."""
    n = l.shape[0]
    big = np.kron(np.eye(n), l) + np.kron(u.T, np.eye(n))
    vec = np.linalg.solve(big, c.flatten(order="F"))
    return vec.reshape((n, n), order="F")
