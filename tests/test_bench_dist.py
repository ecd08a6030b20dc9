"""bench.py's distributed branch on CPU (gloo, world size 2).

`bench.py --gpus 2` without a launcher re-executes itself under
torch.distributed.run with two ranks; `--stub` replaces the kernels by a
rank-dependent sleep so the plumbing (rank setup, per-rank shard, barrier,
max-over-ranks time, whole-job sum, one line from rank 0) runs here.
"""

import json
import socket
import subprocess
import sys
from pathlib import Path

REPO = Path(__file__).resolve().parents[1]


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(args, env_port):
    import os
    env = dict(os.environ, MASTER_PORT=str(env_port), OMP_NUM_THREADS="1")
    env.pop("WORLD_SIZE", None)
    proc = subprocess.run([sys.executable, str(REPO / "bench.py"), *args], capture_output=True, text=True,
                          timeout=300, env=env, cwd=REPO)
    assert proc.returncode == 0, proc.stderr[-2000:]
    lines = [ln for ln in proc.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, proc.stdout
    return json.loads(lines[0])


def test_bench_gpus2_spawns_two_ranks_strong_scaling():
    line = _run(["--gpus", "2", "--stub", "--workload", "c5-chol", "--steps", "3", "--warmup", "3"], _port())
    assert line["n_gpus"] == 2
    assert line["scaling"] == "strong"
    # max over ranks: rank 1 sleeps 2 ms per step
    assert line["ms_per_step"] >= 2.0
    # whole-job flops: 2^20 problems of n = 64 in total, whatever the split
    assert abs(line["value"] * line["ms_per_step"] * 1e-3 * 1e9 - (1 << 20) * 64 ** 3 / 3) < 1e3


def test_bench_single_rank_stub():
    line = _run(["--stub", "--workload", "chol-sweep", "--sizes", "4,8", "--steps", "2", "--warmup", "3"], _port())
    assert line["n_gpus"] == 1 and line["scaling"] == "weak"
