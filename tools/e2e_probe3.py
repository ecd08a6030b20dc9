"""solve_host time per n for Cholesky (banded vs whole copies via LAGEN_HOST_BANDS)."""
import sys, time
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1906_08613_b200 import executor, _lib
torch.cuda.set_device(0)
for n in (16, 32, 48, 64, 96, 128):
    batch = (1 << 28) // (8 * n * n)
    ins = executor.generate("cholesky", n, n, batch)
    host = [t.cpu().pin_memory() for t in ins]
    out = torch.empty_like(host[0]).pin_memory(); info = torch.empty(batch, dtype=torch.int32).pin_memory()
    executor.solve_host("cholesky", host, out=out, info=info)
    ts = []
    for _ in range(3):
        torch.cuda.synchronize(); t = time.perf_counter()
        executor.solve_host("cholesky", host, out=out, info=info)
        ts.append(time.perf_counter() - t)
    h2d, d2h = _lib.host_bytes(0, n, batch)
    print(f"n={n}: solve_host {min(ts)*1e3:.2f} ms, H2D {h2d/1e6:.0f} MB D2H {d2h/1e6:.0f} MB", flush=True)
