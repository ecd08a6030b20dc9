"""CUDA emission from a variant's statement list — the B200 counterpart of the
reference's C back end (`emit_function(build_program(cfg, n))`,
/root/reference/pkg/src/lagen/codegen.py:155-201).

The reference lowers an `Algorithm` (worksheet.py:70-87) at a fixed (n, b) to
a straight-line C function `<eq>_v<k>_n<n>_b<b>(const double* in..., double*
X)` (`_signature`, codegen.py:143-152).  Here the same inputs give a
size-specialised sm_100a kernel: `emit_cuda()` turns the statements — taken
from a live reference `Algorithm`, a built-in `Variant`, or encoded statement
dicts — into one CUDA translation unit that instantiates the warp engine
(`csrc/engine.cuh`: the statement list as a C++ type list, scheduled into
dependency levels at compile time, DMMA block updates, register leaves) for
exactly that (equation, statements, n, b) and exports, C ABI,

    int <name>(const double* in..., double* X, int* info, long long batch, void* stream)

with the inputs in `_signature` order (cholesky: A; lyapunov: L, S;
sylvester: L, U, C), device pointers, row-major ld = n per problem, per-problem
`info` like the library (include/lagen_b200.h), returning a cudaError_t code.
`compile_module()` builds it with nvcc for sm_100a only and `load()` binds it;
`EmittedKernel.solve()` runs it on torch tensors.

This is how every statement list the frontend can synthesise gets a compiled,
fused kernel (the prebuilt library instantiates a measured subset; the generic
engine interprets the rest at run time).  Nothing here falls back to a CPU
path: without nvcc or a CUDA device the calls raise.
"""

import ctypes
import hashlib
import os
import subprocess
import threading
from dataclasses import dataclass
from pathlib import Path

from . import build as _build
from . import errors
from .variants import (EQ_CODES, EQ_INPUTS, Variant, encode_algorithm, stmts_key, validate)

CSRC = _build.CSRC
INCLUDE = _build.INCLUDE
DEFAULT_DIR = _build.PKG / "lib" / "emitted"
_KIND_NAMES = {0: "GEMM_update", 1: "CHOL", 2: "TRSM_left_transposed", 3: "SYLV", 4: "LYAP"}
_OPS = {"cholesky": ("X", "A"), "lyapunov": ("X", "L", "S"), "sylvester": ("X", "L", "U", "C")}


@dataclass(frozen=True)
class EmittedModule:
    name: str        # exported function, <eq>_v<k>_n<n>_b<b>_cuda (or ..._s<hash> for an unnamed list)
    eq: str
    n: int
    b: int
    text: str        # the CUDA translation unit

    @property
    def digest(self):
        return hashlib.sha1(self.text.encode()).hexdigest()[:12]


def _statements(eq, variant):
    """(encoded statements, variant index or None) from a live reference
    Algorithm, a Variant, or statement dicts."""
    if isinstance(variant, Variant):
        return list(variant.statements), variant.index
    if hasattr(variant, "statements") and hasattr(variant, "equation"):
        return encode_algorithm(variant), getattr(variant, "index", None)
    return list(variant), None


def _view(v, trans=None):
    return f"V<{v[0]}, {v[1]}, {v[2]}, {v[3] if trans is None else trans}>"


def _display(eq, s):
    names = _OPS[eq]

    def show(v):
        return f"{names[v[0]]}[{v[1]}][{v[2]}]" + ("^T" if len(v) > 3 and v[3] else "")
    o = show(tuple(s["out"]) + (0,))
    ins = [show(v) for v in s["ins"] if v[0] >= 0]
    if s["kind"] == 0:
        return f"{o} := {o} {'-' if s['sign'] < 0 else '+'} {ins[0]} * {ins[1]}"
    return f"{o} := {_KIND_NAMES[s['kind']]}({', '.join(ins + [o])})"


def emit_cuda(eq, variant, n, b, name=None):
    """One CUDA translation unit for (equation, statement list, n, b)."""
    if eq not in EQ_CODES:
        raise errors.UsageError(f"unknown equation {eq!r}")
    stmts, index = _statements(eq, variant)
    validate(eq, stmts)
    if n < 8 or n > 128 or n % 4:
        raise errors.UnsupportedSizeError("emitted kernels take n in {8, 12, ..., 128}")
    if b not in (4, 8, 16) or n % b:
        raise errors.UnsupportedSizeError(f"block size {b} must be 4, 8 or 16 and divide n = {n}")
    if name is None:
        tag = f"v{index}" if index is not None else "s" + hashlib.sha1(repr(stmts_key(stmts)).encode()).hexdigest()[:8]
        name = f"{eq}_{tag}_n{n}_b{b}_cuda"
    sts = []
    for s in stmts:
        parts = [str(s["kind"]), str(s["sign"]), _view(tuple(s["out"]), 0)]
        parts += [_view(v) for v in s["ins"] if v[0] >= 0]
        sts.append(f"    St<{', '.join(parts)}>  /* {_display(eq, s)} */")
    ins = EQ_INPUTS[eq]
    params = ", ".join(f"const double* {nm}" for nm in ins)
    args = [ins[i] if i < len(ins) else ins[0] for i in range(3)]
    text = f"""// EMITTED by paper_1906_08613_b200/emit.py — {eq}, n = {n}, b = {b}, {len(stmts)} statements.
// Counterpart of the reference's emitted C kernel (codegen.py:155-201) for sm_100a.
#include "registry_warp.cuh"

namespace lagen {{
namespace eng {{
using emitted_var = Var<
{(',' + chr(10)).join(sts)}>;
}}  // namespace eng
}}  // namespace lagen

#define LAGEN_EMIT_API extern "C" __attribute__((visibility("default")))

LAGEN_EMIT_API int {name}({params}, double* X, int* info, long long batch, void* stream) {{
  lagen::LaunchArgs a{{}};
  a.in[0] = {args[0]};
  a.in[1] = {args[1]};
  a.in[2] = {args[2]};
  a.X = X;
  a.info = info;
  a.batch = batch;
  a.prof = nullptr;
  return (int)lagen::launch_warp<{EQ_CODES[eq]}, {n}, {b}, lagen::eng::emitted_var>(a, static_cast<cudaStream_t>(stream));
}}

LAGEN_EMIT_API void {name}_shape(int* eq, int* n, int* b, int* nstmts) {{
  *eq = {EQ_CODES[eq]};
  *n = {n};
  *b = {b};
  *nstmts = {len(stmts)};
}}
"""
    return EmittedModule(name, eq, n, b, text)


def compile_module(mod, out_dir=None, force=False):
    """nvcc -shared for sm_100a; returns the .so path (cached by content hash)."""
    out_dir = Path(out_dir) if out_dir is not None else DEFAULT_DIR
    out_dir.mkdir(parents=True, exist_ok=True)
    so = out_dir / f"{mod.name}.{mod.digest}.so"
    if so.exists() and not force:
        return so
    # per-process / per-thread scratch names: concurrent builds of the same
    # module (two ranks, a thread pool) must not share intermediate files
    uniq = f"{os.getpid()}_{threading.get_ident()}"
    src = out_dir / f"{mod.name}.{mod.digest}.{uniq}.cu"
    src.write_text(mod.text)
    tmp = out_dir / f"{mod.name}.{mod.digest}.{uniq}.tmp"
    # hidden visibility + no STB_GNU_UNIQUE: the module instantiates the same
    # templates as liblagen_b200.so (and as other emitted modules); their
    # function-local statics (per-kernel "configured" flags of launch_warp) and
    # kernel stubs must stay private to each shared object — unique symbols are
    # merged process-wide even under RTLD_LOCAL, and a module would then skip
    # configuring its own copy of the kernel
    cmd = [_build.nvcc(), *_build.ARCH, *_build.NVCC_FLAGS, "-Xcompiler", "-fvisibility=hidden,-fno-gnu-unique",
           f"-I{INCLUDE}", f"-I{CSRC}", "-shared", "-cudart", "static", str(src), "-o", str(tmp)]
    proc = subprocess.run(cmd, capture_output=True, text=True)
    if proc.returncode != 0:
        raise errors.LagenError(f"nvcc failed on the emitted kernel {mod.name}:\n{proc.stderr[-2000:]}")
    os.replace(tmp, so)
    os.replace(src, out_dir / f"{mod.name}.cu")  # keep the last emitted source beside the module
    return so


class EmittedKernel:
    """A loaded emitted module: `solve(inputs) -> (X, info)` on CUDA tensors."""

    def __init__(self, path, name, eq, n, b):
        self.path, self.name, self.eq, self.n, self.b = Path(path), name, eq, n, b
        self._lib = ctypes.CDLL(str(path))
        self._fn = getattr(self._lib, name)
        nin = len(EQ_INPUTS[eq])
        self._fn.argtypes = [ctypes.c_void_p] * (nin + 2) + [ctypes.c_longlong, ctypes.c_void_p]
        self._fn.restype = ctypes.c_int
        shape = getattr(self._lib, name + "_shape")
        vals = [ctypes.c_int() for _ in range(4)]
        shape(*[ctypes.byref(v) for v in vals])
        if (vals[0].value, vals[1].value, vals[2].value) != (EQ_CODES[eq], n, b):
            raise errors.LagenError(f"{path} was emitted for another (equation, n, b)")

    def launch(self, inputs, X, info, stream=None):
        import torch
        batch = X.shape[0]
        for t in list(inputs) + [X]:
            if not (t.is_cuda and t.dtype == torch.float64 and t.is_contiguous() and tuple(t.shape) == (batch, self.n, self.n)):
                raise errors.UsageError("emitted kernels take contiguous float64 CUDA tensors of shape (batch, n, n)")
        if info.dtype != torch.int32 or info.numel() < batch:
            raise errors.UsageError("info must be int32 with one entry per problem")
        stream = stream if stream is not None else torch.cuda.current_stream()
        rc = self._fn(*[t.data_ptr() for t in inputs], X.data_ptr(), info.data_ptr(), batch, stream.cuda_stream)
        if rc != 0:
            raise errors.LagenError(f"emitted kernel {self.name}: CUDA error {rc}")

    def solve(self, inputs):
        import torch
        if len(inputs) != len(EQ_INPUTS[self.eq]):
            raise errors.UsageError(f"{self.eq} takes inputs {EQ_INPUTS[self.eq]}")
        X = torch.empty_like(inputs[0])
        info = torch.zeros(X.shape[0], dtype=torch.int32, device=X.device)
        self.launch(inputs, X, info)
        return X, info


def load(path, mod):
    return EmittedKernel(path, mod.name, mod.eq, mod.n, mod.b)


def compile_variant(eq, variant, n, b, out_dir=None):
    """emit -> nvcc -> load, for a live Algorithm / Variant / statement list."""
    mod = emit_cuda(eq, variant, n, b)
    return load(compile_module(mod, out_dir), mod)


def prebuild(cases, out_dir=None, jobs=None):
    """Emit and compile many (eq, variant, n, b) in parallel (each nvcc run is
    a few seconds); returns the .so paths.  __graft_entry__.build() uses it so
    the emitted-kernel parity tests find their modules in the in-tree cache."""
    from concurrent.futures import ThreadPoolExecutor
    mods = [emit_cuda(eq, v, n, b) for eq, v, n, b in cases]
    jobs = jobs or max(1, min(len(mods), os.cpu_count() or 4))
    with ThreadPoolExecutor(jobs) as ex:
        return list(ex.map(lambda m: compile_module(m, out_dir), mods))
