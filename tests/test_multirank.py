"""Multi-rank sharding logic on CPU (gloo, world_size 2).

The GPU path shards problems by index with no data-path collective
(SURVEY §8e); this test runs the same host logic as bench.py under
torch.distributed with the gloo backend: each rank generates its shard with
the (CPU twin of the) seeded generator, solves it with the oracle executor,
and the gathered result must equal the single-process solve bit for bit;
the max-over-ranks reduction used for timing is exercised too.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1906_08613_b200.shard import shard_range, weak_range


def test_shard_range_covers_exactly():
    for total in (0, 1, 7, 1 << 20):
        for world in (1, 2, 3, 4, 8):
            seen = 0
            nxt = 0
            for r in range(world):
                first, count = shard_range(total, r, world)
                if count:
                    assert first == nxt
                    nxt = first + count
                seen += count
            assert seen == total
    assert weak_range(4096, 3) == (3 * 4096, 4096)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle
    from paper_1906_08613_b200.variants import builtin_variants

    eq, n, total = "sylvester", 12, 10
    first, count = shard_range(total, rank, world)
    ins = oracle.generate(eq, n, 7, first, count)
    X, info = oracle.execute(eq, builtin_variants(eq)[13].statements, n, 4, ins, nthreads=1)
    # gather shards on rank 0 (test only; the GPU path never gathers)
    pad = -(-total // world)
    buf = torch.zeros(pad, n, n, dtype=torch.float64)
    buf[:count] = torch.from_numpy(X)
    bufs = [torch.zeros_like(buf) for _ in range(world)] if rank == 0 else None
    dist.gather(buf, bufs, dst=0)
    t = torch.tensor([float(rank + 1)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        got = torch.cat([b[: shard_range(total, r, world)[1]] for r, b in enumerate(bufs)]).numpy()
        out["X"] = got
        out["max"] = float(t.item())
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gloo_shards_match_single_process():
    from oracle import oracle
    from paper_1906_08613_b200.variants import builtin_variants

    mgr = mp.Manager()
    out = mgr.dict()
    port = _free_port()
    mp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
    eq, n, total = "sylvester", 12, 10
    ins = oracle.generate(eq, n, 7, 0, total)
    X, info = oracle.execute(eq, builtin_variants(eq)[13].statements, n, 4, ins, nthreads=1)
    assert np.array_equal(out["X"], X)
    assert out["max"] == 2.0
