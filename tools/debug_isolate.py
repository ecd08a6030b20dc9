"""Run one small solve per (eq, n, b, variant) in a fresh process and report faults."""
import subprocess, sys
cfgs = []
for eq in ("cholesky", "lyapunov", "sylvester"):
    for n in (4, 8, 16, 32, 64, 128):
        cfgs.append((eq, n))
code = r'''
import sys, torch
sys.path.insert(0, ".")
from paper_1906_08613_b200 import executor
eq, n = sys.argv[1], int(sys.argv[2])
torch.cuda.set_device(0)
A = [torch.eye(n, dtype=torch.float64, device="cuda").expand(3, n, n).contiguous() * (2 + i) for i in range({"cholesky":1,"lyapunov":2,"sylvester":3}[eq])]
X, info = executor.solve(eq, A, variant=0, b=4, check=False)
torch.cuda.synchronize()
print("OK", X[0,0,0].item(), info.tolist())
'''
for eq, n in cfgs:
    p = subprocess.run([sys.executable, "-c", code, eq, str(n)], capture_output=True, text=True,
                       env={**__import__("os").environ, "CUDA_LAUNCH_BLOCKING": "1"}, timeout=120)
    last = (p.stdout.strip().splitlines() or [""])[-1]
    err = [l for l in p.stderr.splitlines() if "Error" in l or "error" in l][-1:] 
    print(eq, n, p.returncode, last, err, flush=True)
