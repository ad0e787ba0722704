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


def launch_plan(gpus: int, environ=None) -> tuple[str, int]:
    """How bench.py runs for `--gpus N`: ("run", N) when the process already belongs to a
    torchrun job of exactly N ranks (or N == 1 without one); ("exec", N) when N > 1 and no
    torchrun environment exists (bench.py then re-executes itself under torch.distributed.run);
    ValueError when a torchrun job's WORLD_SIZE differs from N (a silent 1-GPU number
    reported as N GPUs is what this prevents)."""
    environ = os.environ if environ is None else environ
    if gpus < 1:
        raise ValueError(f"--gpus must be >= 1, got {gpus}")
    if "WORLD_SIZE" in environ:
        ws = int(environ["WORLD_SIZE"])
        if ws != gpus:
            raise ValueError(f"--gpus {gpus} but the torchrun job has WORLD_SIZE={ws}")
        return "run", ws
    return ("exec", gpus) if gpus > 1 else ("run", 1)


def torchrun_argv(python: str, script: str, gpus: int, port: int, args: list[str]) -> list[str]:
    """argv of the one-node torchrun launch (127.0.0.1 rendezvous, one rank per GPU)."""
    return [python, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={gpus}",
            "--master-addr=127.0.0.1", f"--master-port={port}", script, *args]


def sample_indices(n_total: int, m: int, offset: int, count: int):
    """The accuracy sample (bench.py max_ulp_err): m evenly spaced global indices over
    [0, n_total), restricted to this rank's slice [offset, offset + count) and returned as local
    indices.  The union over ranks is the same sample for every world size."""
    import numpy as np
    if n_total <= 0 or m <= 0:
        return np.zeros(0, np.int64)
    g = np.unique(np.linspace(0, n_total - 1, min(m, n_total)).astype(np.int64))
    g = g[(g >= offset) & (g < offset + count)]
    return g - offset


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


def reduce_accuracy(worst, sums):
    """MAX of the per-rank maximum errors and SUM of the per-rank sample counts/violations
    (float64 tensors), in place; no-op without a process group."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized():
        dist.all_reduce(worst, op=dist.ReduceOp.MAX)
        dist.all_reduce(sums, op=dist.ReduceOp.SUM)
    return worst, sums


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
