import time, sys, torch
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1906_08613_b200 import executor
torch.cuda.set_device(0)
for eq, n in (("cholesky", 64), ("cholesky", 16), ("sylvester", 64)):
    batch = (1 << 28) // (8 * n * n)
    ins = executor.generate(eq, n, n, batch)
    host = [t.cpu().pin_memory() for t in ins]
    out = torch.empty_like(host[0]).pin_memory(); info = torch.empty(batch, dtype=torch.int32).pin_memory()
    executor.solve_host(eq, host, out=out, info=info)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(3):
        executor.solve_host(eq, host, out=out, info=info)
    dt = (time.perf_counter() - t0) / 3
    byt = sum(t.numel() * 8 for t in host) + out.numel() * 8
    t1 = time.perf_counter()
    for _ in range(3):
        for h, d in zip(host, ins):
            d.copy_(h, non_blocking=True)
        out.copy_(ins[0], non_blocking=True)
    torch.cuda.synchronize()
    dc = (time.perf_counter() - t1) / 3
    print(f"{eq} n={n}: solve_host {dt*1e3:.1f} ms ({byt/dt/1e9:.1f} GB/s moved); plain copies {dc*1e3:.1f} ms ({byt/dc/1e9:.1f} GB/s)")
