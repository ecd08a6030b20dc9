"""Where does the host-pipeline time go? (chol n=16 vs n=64)"""
import sys, time
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1906_08613_b200 import executor
torch.cuda.set_device(0)
for n in (16, 64):
    batch = (1 << 28) // (8 * n * n)
    ins = executor.generate("cholesky", n, n, batch)
    host = [t.cpu().pin_memory() for t in ins]
    out = torch.empty_like(host[0]).pin_memory(); info = torch.empty(batch, dtype=torch.int32).pin_memory()
    for eng in ("column", "generic", "rows", "auto"):
        try:
            executor.solve_host("cholesky", host, variant=1, b=4, out=out, info=info, engine=eng)
        except Exception as e:
            print(n, eng, "n/a", e); continue
        torch.cuda.synchronize(); t = time.perf_counter()
        executor.solve_host("cholesky", host, variant=1, b=4, out=out, info=info, engine=eng)
        dt = time.perf_counter() - t
        chunk = (16 << 20) // (8 * n * n)
        X = torch.empty_like(ins[0]); inf = torch.empty(batch, dtype=torch.int32, device="cuda")
        sub = [t[:chunk] for t in ins]
        executor.solve("cholesky", sub, variant=1, b=4, out=X[:chunk], info=inf[:chunk], engine=eng, check=False)
        torch.cuda.synchronize(); t2 = time.perf_counter()
        for _ in range(10):
            executor.solve("cholesky", sub, variant=1, b=4, out=X[:chunk], info=inf[:chunk], engine=eng, check=False)
        torch.cuda.synchronize(); dk = (time.perf_counter() - t2) / 10
        print(f"n={n} {eng}: solve_host {dt*1e3:.1f} ms; one chunk ({chunk}) device solve {dk*1e3:.3f} ms", flush=True)
