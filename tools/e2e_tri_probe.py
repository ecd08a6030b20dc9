"""Host-path time per n: dense staged copies vs zero-copy triangles (and the
caller-zeroed X), Cholesky batches of 256 MiB, pinned buffers."""
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1906_08613_b200 import executor  # noqa: E402

eq = sys.argv[1] if len(sys.argv) > 1 else "cholesky"
for n in (8, 16, 32, 64, 96, 128):
    batch = (1 << 28) // (8 * n * n)
    ins = executor.generate(eq, n, seed=n, batch=batch)
    host = [t.cpu().pin_memory() for t in ins]
    out = torch.zeros((batch, n, n), dtype=torch.float64).pin_memory()
    info = torch.empty(batch, dtype=torch.int32).pin_memory()
    row = []
    for tri, z in ((False, False), (True, False), (True, eq == "cholesky")):
        executor.solve_host(eq, host, out=out, info=info, triangles=tri, out_zeroed=z)
        t0 = time.perf_counter()
        for _ in range(3):
            executor.solve_host(eq, host, out=out, info=info, triangles=tri, out_zeroed=z)
        row.append((time.perf_counter() - t0) / 3 * 1e3)
    print(f"{eq} n={n}: dense {row[0]:.2f} ms  triangles {row[1]:.2f} ms  triangles+zeroed {row[2]:.2f} ms", flush=True)
