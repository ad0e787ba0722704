"""Multi-GPU plumbing for the arc/latitude path: one process per GPU, `torch.distributed`.

The path partitions into independent queries, so ranks own disjoint
slices of the global index space and there is no data-path collective.  The only exchanges are
after the timed region: the step time (MAX over ranks, the driver's timing rule) and the count
histogram (SUM), both tiny tensors over NCCL (GPU) or gloo (CPU tests).
"""
from __future__ import annotations

import os


def env() -> tuple[int, int, int]:
    """(world_size, rank, local_rank) from the torchrun environment (1, 0, 0 when absent)."""
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


def shard_weak(rank: int, world: int, n_per_rank: int) -> tuple[int, int]:
    """Weak scaling: rank r owns global indices [r*n, (r+1)*n) -> (offset, count)."""
    if not 0 <= rank < world or n_per_rank < 0:
        raise ValueError("bad shard arguments")
    return rank * n_per_rank, n_per_rank


def shard_strong(rank: int, world: int, n_total: int) -> tuple[int, int]:
    """Strong scaling: rank r owns [floor(r*N/R), floor((r+1)*N/R)) -> (offset, count)."""
    if not 0 <= rank < world or n_total < 0:
        raise ValueError("bad shard arguments")
    lo, hi = rank * n_total // world, (rank + 1) * n_total // world
    return lo, hi - lo


def reduce_after_step(elapsed_ms, hist, stats=None, counts=None):
    """MAX of the per-rank step time and SUM of the count histograms (in place; returns them);
    optionally MAX of the output statistics and SUM of their violation counts
    (sgi_output_stats: SURVEY §8(e) "NCCL reduction of counts and max-ulp statistics").

    `elapsed_ms` is a float64 tensor of shape (1,), `hist` an int64 tensor of shape (5,),
    `stats` float64 and `counts` int64 tensors, all on the process group's device (CUDA for
    NCCL, CPU for gloo).  No-op without a process group."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized():
        dist.all_reduce(elapsed_ms, op=dist.ReduceOp.MAX)
        dist.all_reduce(hist, op=dist.ReduceOp.SUM)
        if stats is not None:
            dist.all_reduce(stats, op=dist.ReduceOp.MAX)
        if counts is not None:
            dist.all_reduce(counts, op=dist.ReduceOp.SUM)
    if stats is None and counts is None:
        return elapsed_ms, hist
    return elapsed_ms, hist, stats, counts
