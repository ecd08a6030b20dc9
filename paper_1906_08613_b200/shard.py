"""Problem-index sharding across GPUs.

Problems are independent, so a batch shards by contiguous index range with
no data-path collective.  Every problem's inputs are a pure function of
(seed, equation, n, global index) (generate.cu), so any sharding sees the
same problems; torch.distributed is used only for the start/stop barrier and
the max-over-ranks device time.
"""


def shard_range(total, rank, world):
    """Contiguous range [first, first + count) of `total` problems for `rank`
    (ceil-divided, the last ranks may get fewer or none)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    per = -(-total // world)
    first = min(total, rank * per)
    count = max(0, min(total, first + per) - first)
    return first, count


def weak_range(batch_per_rank, rank):
    """Weak scaling: each rank solves its own batch of fresh problems."""
    return rank * batch_per_rank, batch_per_rank
