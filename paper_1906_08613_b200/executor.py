"""Host-side executor API: the reference's hot-path interface backed by the
sm_100a kernels.

Reference interface being replaced:
  * interpret_algorithm(alg, inst, b, on_iteration=None) -> ({X: ndarray}, flops)
      /root/reference/pkg/src/lagen/verify.py:221-303
  * the emitted kernel <eq>_v<k>_n<n>_b<b>(inputs..., X)
      /root/reference/pkg/src/lagen/codegen.py:155-201
Batched additions:
  * solve(eq, inputs, variant=..., b=...) on [batch, n, n] fp64 CUDA tensors
  * execute_batched(alg, n, b, {name: tensor}) -> {X: tensor}
  * solve_host(...) for host (numpy / pinned) buffers through the pipelined
    C entry point
  * generate(eq, n, seed, batch, first) — the seeded batched generator.

Everything runs on the GPU through liblagen_b200.so; there is no CPU path.
"""

import ctypes

import numpy as np
import torch

from . import _lib, dispatch, errors
from .variants import (EQ_CODES, EQ_INPUTS, EQUATIONS, Variant, builtin_variants,
                       classify_equation, encode_algorithm, flop_count, validate)


def _eq_name(eq):
    if isinstance(eq, str):
        if eq not in EQUATIONS:
            # accept the reference's short names (verify.classify)
            short = {"chol": "cholesky", "lyap": "lyapunov", "sylv": "sylvester"}
            if eq in short:
                return short[eq]
            raise errors.UsageError(f"unknown equation {eq!r}")
        return eq
    if isinstance(eq, int):
        return EQUATIONS[eq]
    return classify_equation(eq)


def resolve_variant(eq_name, variant):
    """variant: None (dispatch), int index, Variant, reference Algorithm, or a
    list of encoded statement dicts.  Returns (stmts, variant_index_or_None)."""
    if variant is None:
        return None, None
    if isinstance(variant, int):
        vs = builtin_variants(eq_name)
        if not 0 <= variant < len(vs):
            raise errors.VariantError(f"{eq_name} has {len(vs)} variants, not {variant}")
        return vs[variant].statements, variant
    if isinstance(variant, Variant):
        return variant.statements, variant.index
    if hasattr(variant, "statements") and hasattr(variant, "equation"):
        return encode_algorithm(variant), getattr(variant, "index", None)
    return list(variant), None


def _resolve(eq_name, n, variant, b, engine):
    """(stmts, variant_index, b, engine) for a solve: the dispatch table's
    measured (variant, b, engine) fills what the caller left open.  The
    table's engine is used only when it runs the requested (variant, b)
    (it was chosen for the table's b); otherwise "auto"."""
    stmts, idx = resolve_variant(eq_name, variant)
    pick = dispatch.select(eq_name, n)
    if stmts is None:
        idx = pick["variant"]
        stmts = builtin_variants(eq_name)[idx].statements
    if b is None:
        b = pick["b"]
    if engine is None:
        engine = "auto"
        table_engine = pick.get("engine") or "auto"
        if idx is not None and idx == pick["variant"] and table_engine != "auto":
            if b == pick["b"] or _lib.engine_supported(EQ_CODES[eq_name], n, b, idx, table_engine):
                engine = table_engine
    if engine not in _lib.ENGINES and engine != EMITTED:
        raise errors.UsageError(f"unknown engine {engine!r}; one of {sorted(_lib.ENGINES) + [EMITTED]}")
    return stmts, idx, b, engine


# engine "emitted": the statement list is emitted as its own size-specialised
# CUDA kernel (emit.py, the counterpart of the reference's emit_function),
# compiled with nvcc on first use and cached on disk and in the process
EMITTED = "emitted"
_emitted = {}


def _emitted_kernel(eq_name, stmts, idx, n, b):
    from . import emit
    from .variants import stmts_key
    key = (eq_name, stmts_key(stmts), n, b)
    k = _emitted.get(key)
    if k is None:
        variant = builtin_variants(eq_name)[idx] if idx is not None else stmts
        k = _emitted[key] = emit.compile_variant(eq_name, variant, n, b)
    return k


def _stream_ptr(stream):
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


def _check_inputs(eq_name, inputs, n=None):
    names = EQ_INPUTS[eq_name]
    if len(inputs) != len(names):
        raise errors.UsageError(f"{eq_name} takes inputs {names}, got {len(inputs)} tensors")
    shape = None
    for nm, t in zip(names, inputs):
        if not isinstance(t, torch.Tensor):
            raise errors.UsageError(f"input {nm} must be a torch.Tensor")
        if t.dtype != torch.float64:
            raise errors.UsageError(f"input {nm} must be float64, got {t.dtype}")
        if not t.is_cuda:
            raise errors.UsageError(f"input {nm} must live on a CUDA device")
        if t.dim() != 3 or t.shape[1] != t.shape[2]:
            raise errors.UsageError(f"input {nm} must be [batch, n, n], got {tuple(t.shape)}")
        if not t.is_contiguous():
            raise errors.UsageError(f"input {nm} must be contiguous (row-major, ld = n)")
        if shape is None:
            shape = tuple(t.shape)
        elif tuple(t.shape) != shape:
            raise errors.UsageError("inputs disagree in shape")
    if n is not None and shape[1] != n:
        raise errors.UsageError(f"inputs are {shape[1]}x{shape[1]}, expected n={n}")
    return shape[0], shape[1]


def solve(eq, inputs, variant=None, b=None, out=None, info=None, stream=None, check=True, engine=None):
    """Solve a batch: inputs in _signature order (chol: A; lyap: L, S;
    sylv: L, U, C), each [batch, n, n] float64 CUDA contiguous.

    variant/b default to the dispatch table (the GPU analogue of cli._select).
    Returns (X, info).  With check=True a non-zero info raises
    VerificationError like the reference (kernels.py:87-88, verify.py:301-302);
    that forces a device sync."""
    eq_name = _eq_name(eq)
    batch, n = _check_inputs(eq_name, inputs)
    stmts, idx, b, engine = _resolve(eq_name, n, variant, b, engine)
    validate(eq_name, stmts)
    dev = inputs[0].device
    if out is None:
        out = torch.empty((batch, n, n), dtype=torch.float64, device=dev)
    if info is None:
        info = torch.empty(batch, dtype=torch.int32, device=dev)
    if engine == EMITTED:
        with torch.cuda.device(dev):
            _emitted_kernel(eq_name, stmts, idx, n, b).launch(inputs, out, info, stream)
    else:
        arr = _lib.stmt_array(stmts)
        ptrs = (ctypes.c_void_p * 3)(*([t.data_ptr() for t in inputs] + [0] * (3 - len(inputs))))
        with torch.cuda.device(dev):
            rc = _lib.lib.lagen_b200_execute_engine(EQ_CODES[eq_name], ctypes.addressof(arr), len(stmts), n, b,
                                                    batch, ctypes.addressof(ptrs), ctypes.c_void_p(out.data_ptr()),
                                                    ctypes.c_void_p(info.data_ptr()), _stream_ptr(stream),
                                                    _lib.ENGINES[engine])
        _lib.check(rc, f"{eq_name} n={n} b={b} engine={engine}")
    if check and batch:
        bad = torch.nonzero(info).flatten()
        if bad.numel():
            p = int(bad[0])
            code = int(info[p])
            if code > 0:
                raise errors.VerificationError(f"problem {p}: non-positive pivot at index {code - 1}")
            raise errors.VerificationError(f"problem {p}: NaN or Inf produced: ill-posed instance or bug")
    return out, info


class Plan:
    """A prepared batched solve: arguments marshalled once, launched many
    times (no per-call validation or allocation) — suitable for CUDA-graph
    capture of a whole sweep."""

    def __init__(self, eq, inputs, variant=None, b=None, out=None, info=None, engine=None):
        self.eq = _eq_name(eq)
        self.batch, self.n = _check_inputs(self.eq, inputs)
        stmts, idx, b, engine = _resolve(self.eq, self.n, variant, b, engine)
        validate(self.eq, stmts)
        self.variant, self.b, self.stmts = idx, b, stmts
        self.engine = engine
        dev = inputs[0].device
        self.inputs = list(inputs)
        self.out = out if out is not None else torch.empty((self.batch, self.n, self.n),
                                                           dtype=torch.float64, device=dev)
        self.info = info if info is not None else torch.empty(self.batch, dtype=torch.int32, device=dev)
        self._arr = _lib.stmt_array(stmts)
        self._ptrs = (ctypes.c_void_p * 3)(*([t.data_ptr() for t in inputs] + [0] * (3 - len(inputs))))
        self._args = (EQ_CODES[self.eq], ctypes.addressof(self._arr), len(stmts), self.n, b, self.batch,
                      ctypes.addressof(self._ptrs), ctypes.c_void_p(self.out.data_ptr()),
                      ctypes.c_void_p(self.info.data_ptr()))
        self.device = dev
        self._kernel = _emitted_kernel(self.eq, stmts, idx, self.n, b) if engine == EMITTED else None

    def launch(self, stream=None):
        if self._kernel is not None:
            self._kernel.launch(self.inputs, self.out, self.info, stream)
            return self.out
        rc = _lib.lib.lagen_b200_execute_engine(*self._args, _stream_ptr(stream), _lib.ENGINES[self.engine])
        _lib.check(rc, f"{self.eq} n={self.n} b={self.b}")
        return self.out


def execute_batched(alg, n, b, inputs, stream=None, check=True):
    """SURVEY §8b Python side: semantics of interpret_algorithm over a batch.

    alg: reference Algorithm, Variant, or (eq_name, variant_index);
    inputs: {operand name: [batch, n, n] CUDA tensor}.  Returns {X: tensor}."""
    if isinstance(alg, tuple):
        eq_name, alg = alg
    elif isinstance(alg, Variant):
        eq_name = alg.equation
    else:
        eq_name = _eq_name(alg.equation)
    tensors = [inputs[nm] for nm in EQ_INPUTS[eq_name]]
    _check_inputs(eq_name, tensors, n)
    X, _ = solve(eq_name, tensors, variant=alg, b=b, stream=stream, check=check)
    return {"X": X}


def interpret_algorithm(alg, inst, b, on_iteration=None):
    """Drop-in for verify.interpret_algorithm (verify.py:221-303) on one
    reference Instance, executed by the CUDA kernel.  Returns
    ({X: ndarray}, flops) with flops from the reference's exact model."""
    if on_iteration is not None:
        raise errors.UsageError("on_iteration hooks need the per-iteration interpreter; "
                                "the fused CUDA kernel has no iteration boundary")
    eq_name = _eq_name(alg.equation)
    n = inst.n
    if n % b:
        raise errors.VerificationError(f"block size {b} does not divide {n}")
    dev = torch.device("cuda", torch.cuda.current_device())
    tensors = [torch.from_numpy(np.ascontiguousarray(inst.bindings[nm], dtype=np.float64))
               .reshape(1, n, n).to(dev) for nm in EQ_INPUTS[eq_name]]
    X, _ = solve(eq_name, tensors, variant=alg, b=b)
    stmts, _ = resolve_variant(eq_name, alg)
    return {alg.output: X[0].cpu().numpy()}, flop_count(eq_name, stmts, n, b)


def host_triangles_default(eq_name, n):
    """Whether solve_host moves triangles only by default: measured per n
    (tools/e2e_probe4.py, profiles/r02_e2e_hybrid.txt) the hybrid transfer —
    copy engines for the contiguous mostly-needed half of each triangular
    operand, zero-copy kernels for the remaining small triangle — beats dense
    copies from n = 16 on for all three equations (n even, n <= 128)."""
    return 16 <= n <= 128 and n % 2 == 0


_pending_host = []  # host buffers of queued wait=False calls, kept alive until host_sync()


def host_sync():
    """Wait for every queued `solve_host(..., wait=False)` call of the current
    device (lagen_b200_host_sync); their X / info are valid afterwards."""
    rc = _lib.lib.lagen_b200_host_sync()
    _pending_host.clear()
    _lib.check(rc, "host pipeline sync")


def solve_host(eq, inputs, variant=None, b=None, out=None, info=None, engine=None, triangles=None,
               out_zeroed=False, wait=True):
    """Host buffers (numpy arrays or CPU tensors, ideally pinned) -> host X.
    Streams the batch through the GPU with transfer / solve overlap; runs the
    same kernel as solve() (dispatch-table engine unless given).

    triangles: move only the structurally needed part of each operand over
    PCIe (zero-copy kernels on the mapped pinned buffers, LAGEN_HOST_TRIANGLES).
    The copy engines move the contiguous, mostly-needed half of the rows of
    each triangular operand (one strided copy per chunk) and zero-copy kernels
    the remaining small triangle (the engines sustain ~45 GB/s each way under
    bidirectional load, the kernels ~25); the default (None) does this from
    n = 16 on (host_triangles_default; pinned buffers, even n).  out_zeroed: `out`
    already holds zeros in X's structurally-zero part — the reference's own
    contract for its emitted kernels (codegen.py:4-7) — so Cholesky writes
    only X's upper triangle (LAGEN_HOST_X_ZEROED).  wait=False queues the
    call and returns (LAGEN_HOST_ASYNC): a sequence of batches then shares one
    pipeline fill / drain; call host_sync() before reading X or info and keep
    the input buffers untouched until then."""
    eq_name = _eq_name(eq)
    if out_zeroed and out is None:
        raise errors.UsageError("out_zeroed needs a caller-provided out buffer")
    names = EQ_INPUTS[eq_name]
    if len(inputs) != len(names):
        raise errors.UsageError(f"{eq_name} takes inputs {names}, got {len(inputs)} arrays")
    arrs = []
    for nm, t in zip(names, inputs):
        if isinstance(t, torch.Tensor):
            if t.is_cuda or t.dtype != torch.float64 or not t.is_contiguous():
                raise errors.UsageError(f"host input {nm} must be a contiguous float64 CPU tensor")
            arrs.append(t)
        else:
            a = np.ascontiguousarray(t, dtype=np.float64)
            arrs.append(torch.from_numpy(a))
    shape = tuple(arrs[0].shape)
    if len(shape) != 3 or shape[1] != shape[2]:
        raise errors.UsageError(f"host inputs must be [batch, n, n], got {shape}")
    if any(tuple(a.shape) != shape for a in arrs):
        raise errors.UsageError("host inputs disagree in shape")
    batch, n = shape[0], shape[1]
    stmts, idx, b, engine = _resolve(eq_name, n, variant, b, engine)
    validate(eq_name, stmts)
    if out is None:
        out = torch.empty((batch, n, n), dtype=torch.float64, pin_memory=arrs[0].is_pinned())
    elif (not isinstance(out, torch.Tensor) or out.is_cuda or out.dtype != torch.float64
          or tuple(out.shape) != shape or not out.is_contiguous()):
        raise errors.UsageError(f"out must be a contiguous float64 CPU tensor of shape {shape}")
    if info is None:
        info = torch.empty(batch, dtype=torch.int32)
    elif (not isinstance(info, torch.Tensor) or info.is_cuda or info.dtype != torch.int32
          or info.numel() < batch or not info.is_contiguous()):
        raise errors.UsageError(f"info must be a contiguous int32 CPU tensor with >= {batch} entries")
    arr = _lib.stmt_array(stmts)
    ptrs = (ctypes.c_void_p * 3)(*([t.data_ptr() for t in arrs] + [0] * (3 - len(arrs))))
    if triangles is None:
        triangles = (host_triangles_default(eq_name, n) and all(a.is_pinned() for a in arrs)
                     and out.is_pinned())
    flags = ((_lib.HOST_TRIANGLES if triangles else 0) | (_lib.HOST_X_ZEROED if out_zeroed else 0)
             | (0 if wait else _lib.HOST_ASYNC))
    if not wait:
        _pending_host.append((arrs, out, info))
    rc = _lib.lib.lagen_b200_execute_host_flags(EQ_CODES[eq_name], ctypes.addressof(arr), len(stmts), n, b,
                                                batch, ctypes.addressof(ptrs), ctypes.c_void_p(out.data_ptr()),
                                                ctypes.c_void_p(info.data_ptr()), _lib.ENGINES[engine], flags)
    _lib.check(rc, f"{eq_name} host n={n} b={b}")
    return out, info


def generate(eq, n, seed, batch, first=0, device=None, stream=None):
    """Seeded batched inputs (BASELINE.json distributions) for problems
    [first, first + batch); returns tensors in _signature order."""
    eq_name = _eq_name(eq)
    dev = device or torch.device("cuda", torch.cuda.current_device())
    outs = [torch.empty((batch, n, n), dtype=torch.float64, device=dev) for _ in EQ_INPUTS[eq_name]]
    ptrs = (ctypes.c_void_p * 3)(*([t.data_ptr() for t in outs] + [0] * (3 - len(outs))))
    with torch.cuda.device(dev):
        rc = _lib.lib.lagen_b200_generate(EQ_CODES[eq_name], n, seed, first, batch,
                                          ctypes.addressof(ptrs), _stream_ptr(stream))
    _lib.check(rc, "generate")
    return outs
