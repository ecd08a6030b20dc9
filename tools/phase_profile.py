"""Cycle accounting of one warp-engine problem group (clock64 per phase and
per schedule level), to see where a problem's time goes.

    python tools/phase_profile.py --eq cholesky --n 128 --variant 1 --b 8
"""
import argparse, ctypes, sys
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1906_08613_b200 import _lib, executor
from paper_1906_08613_b200.variants import EQ_CODES, builtin_variants

ap = argparse.ArgumentParser()
ap.add_argument("--eq", default="cholesky"); ap.add_argument("--n", type=int, default=128)
ap.add_argument("--variant", type=int, default=1); ap.add_argument("--b", type=int, default=8)
a = ap.parse_args()
torch.cuda.set_device(0)
batch = (1 << 28) // (8 * a.n * a.n)
ins = executor.generate(a.eq, a.n, a.n, batch)
X = torch.empty_like(ins[0]); info = torch.empty(batch, dtype=torch.int32, device="cuda")
prof = torch.zeros(32, dtype=torch.int64, device="cuda")
st = builtin_variants(a.eq)[a.variant].statements
arr = _lib.stmt_array(st)
ptrs = (ctypes.c_void_p * 3)(*([t.data_ptr() for t in ins] + [0] * (3 - len(ins))))
args = lambda p: (EQ_CODES[a.eq], ctypes.addressof(arr), len(st), a.n, a.b, batch, ctypes.addressof(ptrs),
                  ctypes.c_void_p(X.data_ptr()), ctypes.c_void_p(info.data_ptr()),
                  ctypes.c_void_p(torch.cuda.current_stream().cuda_stream), 2, ctypes.c_void_p(p))
_lib.check(_lib.lib.lagen_b200_execute_profile(*args(0)), "warm")
torch.cuda.synchronize()
_lib.check(_lib.lib.lagen_b200_execute_profile(*args(prof.data_ptr())), "prof")
torch.cuda.synchronize()
p = prof.cpu().tolist()
nprob = max(1, p[3])
print(f"{a.eq} n={a.n} v{a.variant} b{a.b}: problems={p[3]} cycles/problem: wait={p[0]/nprob:.0f} "
      f"compute={p[1]/nprob:.0f} store={p[2]/nprob:.0f}  levels=" +
      " ".join(f"L{i}:{p[4+i]/nprob:.0f}" for i in range(8) if p[4 + i]))
for i, stmt in enumerate(st[:10]):
    print(f"  s{i} {stmt['kind']}->{tuple(stmt['out'])}: warp0 {p[12+i]/nprob:.0f}  warp1 {p[22+i]/nprob:.0f}")
