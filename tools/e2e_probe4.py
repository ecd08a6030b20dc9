"""Host-path rates per n (Cholesky sweep batches): dense staged copies vs
zero-copy triangles (+ caller-zeroed X), queued (wait=False) in groups of 4
calls so pipeline fill / drain is amortised like in bench.py, against a plain
bidirectional chunked copy of the same dense bytes."""
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1906_08613_b200 import _lib, executor  # noqa: E402
from paper_1906_08613_b200.variants import EQ_CODES  # noqa: E402

eq = sys.argv[1] if len(sys.argv) > 1 else "cholesky"
torch.cuda.set_device(0)
# plain bidirectional copy baseline: 256 MiB each way, 16 MiB chunks, 4 streams
nb = 1 << 28
h_in = torch.empty(nb, dtype=torch.uint8).pin_memory()
h_out = torch.empty(nb, dtype=torch.uint8).pin_memory()
d = [torch.empty(1 << 24, dtype=torch.uint8, device="cuda") for _ in range(4)]
st = [torch.cuda.Stream() for _ in range(4)]
def bidi():
    for i in range(nb >> 24):
        k = i % 4
        with torch.cuda.stream(st[k]):
            d[k].copy_(h_in[i << 24:(i + 1) << 24], non_blocking=True)
            h_out[i << 24:(i + 1) << 24].copy_(d[k], non_blocking=True)
    torch.cuda.synchronize()
bidi()
t0 = time.perf_counter()
for _ in range(4):
    bidi()
dt = (time.perf_counter() - t0) / 4
print(f"plain bidirectional copy: {nb / dt / 1e9:.1f} GB/s each way ({dt * 1e3:.2f} ms per 256 MiB)", flush=True)
del h_in, h_out
for n in (8, 16, 32, 40, 48, 56, 64, 80, 96, 112, 128):
    batch = (1 << 28) // (8 * n * n)
    ins = executor.generate(eq, n, seed=n, batch=batch)
    host = [t.cpu().pin_memory() for t in ins]
    outs = [torch.zeros((batch, n, n), dtype=torch.float64).pin_memory() for _ in range(2)]
    info = torch.empty(batch, dtype=torch.int32).pin_memory()
    row = []
    for tri, z in ((False, False), (True, eq == "cholesky")):
        def go():
            for r in range(4):
                executor.solve_host(eq, host, out=outs[r % 2], info=info, triangles=tri, out_zeroed=z, wait=False)
            executor.host_sync()
        go()
        t0 = time.perf_counter()
        go()
        ms = (time.perf_counter() - t0) / 4 * 1e3
        fl = (_lib.HOST_TRIANGLES if tri else 0) | (_lib.HOST_X_ZEROED if z else 0)
        h2d, d2h = _lib.host_bytes(EQ_CODES[eq], n, batch, fl)
        row.append(f"{ms:.2f} ms ({h2d / ms / 1e6:.1f} / {d2h / ms / 1e6:.1f} GB/s in/out)")
    print(f"{eq} n={n}: dense {row[0]}   triangles {row[1]}", flush=True)
