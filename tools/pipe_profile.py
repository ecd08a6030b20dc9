"""Per-step clock64 timeline of one pipe-engine problem (CTA 0's first
problem): solver warp 0 (start, after the critical DMMAs, after the solve,
after the write-out) and updater warp 0 (start, end) per anti-diagonal step.

    python tools/pipe_profile.py --eq sylvester --n 128

The stamps are compiled out of the default library (they cost ~4 % of the
kernel's instructions); build it with them first:

    LAGEN_NVCC_EXTRA=-DLAGEN_PIPE_PROF=1 python -m paper_1906_08613_b200.build --force

(or use tools/experiments/pipe_bench.cu, which tools/experiments/pipe_build.sh
builds with the stamps).
"""
import argparse
import ctypes
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1906_08613_b200 import _lib, executor  # noqa: E402
from paper_1906_08613_b200.variants import EQ_CODES, builtin_variants  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--eq", default="sylvester")
ap.add_argument("--n", type=int, default=128)
a = ap.parse_args()
torch.cuda.set_device(0)
v = 13 if a.eq == "sylvester" else 5
batch = (1 << 28) // (8 * a.n * a.n)
ins = executor.generate(a.eq, a.n, a.n, batch)
X = torch.empty_like(ins[-1])
info = torch.empty(batch, dtype=torch.int32, device="cuda")
prof = torch.zeros(512, dtype=torch.int64, device="cuda")
st = builtin_variants(a.eq)[v].statements
arr = _lib.stmt_array(st)
ptrs = (ctypes.c_void_p * 3)(*([t.data_ptr() for t in ins] + [0] * (3 - len(ins))))


def run(p):
    _lib.check(_lib.lib.lagen_b200_execute_profile(
        EQ_CODES[a.eq], ctypes.addressof(arr), len(st), a.n, 8 if a.n % 8 == 0 else 4, batch,
        ctypes.addressof(ptrs), ctypes.c_void_p(X.data_ptr()), ctypes.c_void_p(info.data_ptr()),
        ctypes.c_void_p(torch.cuda.current_stream().cuda_stream), _lib.ENGINES["pipe"], ctypes.c_void_p(p)), "run")


run(0)
torch.cuda.synchronize()
run(prof.data_ptr())
torch.cuda.synchronize()
p = prof.cpu().tolist()
T = (a.n + 7) // 8
t0 = min(x for x in p if x) if any(p) else 0
print(f"{a.eq} n={a.n} T={T}: per step (cycles from the first stamp)")
print(" d   sol:start handover solve out | upd:start end")
prev = None
for d in range(-1, 2 * T - 1):
    s = p[4 * (d + 1): 4 * (d + 1) + 4]
    u = p[256 + 2 * (d + 1): 256 + 2 * (d + 1) + 2]
    f = lambda x: f"{x - t0:7d}" if x else "      -"
    dur = f"wait={s[1]-s[0]} solve={s[2]-s[1]} out={s[3]-s[2]}" if all(s) else ""
    ud = f"upd={u[1]-u[0]}" if all(u) else ""
    print(f"{d:2d} {f(s[0])} {f(s[1])} {f(s[2])} {f(s[3])} | {f(u[0])} {f(u[1])}   {dur} {ud}")
