"""Multi-process (gloo, world size 2, CPU) test of the sharding and the post-step reduction used
by bench.py's torchrun path: the shards' union is the global index range, and the reduced
histogram equals the single-process one (the hot path is replaced by oracle (a) on CPU; the GPU
kernel's R-invariance is tested separately in test_gpu_parity.py)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import sgi_inputs
from paper_2510_09892_b200 import dist as sdist


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _hist(cnt):
    return np.array([(cnt == 0).sum(), (cnt == 1).sum(), (cnt == 2).sum(), (cnt == 0xFF).sum(),
                     (cnt == 1).sum() + 2 * (cnt == 2).sum()], np.int64)


def _worker(rank, world, port, n_per_rank, config, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ws, r, _ = sdist.env()
    off, cnt_n = sdist.shard_weak(r, ws, n_per_rank)
    a, b, z0 = sgi_inputs.generate_host(config, cnt_n, offset=off)
    _, cnt = oracle.intersect(oracle.MODE_EFT, a, b, z0)
    hist = torch.from_numpy(_hist(cnt))
    t = torch.tensor([10.0 + r], dtype=torch.float64)
    stats = torch.tensor([0.5 + r, 2.0 - r], dtype=torch.float64)
    counts = torch.tensor([r, 2 * r], dtype=torch.int64)
    t, hist, stats, counts = sdist.reduce_after_step(t, hist, stats, counts)
    q.put((r, float(t.item()), hist.numpy().tolist(), stats.tolist(), counts.tolist()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("config", [5, 3])
def test_gloo_world2_sharded_histogram(config):
    world, n = 2, 3000
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, config, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    a, b, z0 = sgi_inputs.generate_host(config, world * n)
    _, cnt = oracle.intersect(oracle.MODE_EFT, a, b, z0)
    want = _hist(cnt).tolist()
    for r, t, h, st, ct in res:
        assert t == 11.0                       # MAX over ranks
        assert h == want                       # SUM of shard histograms == global histogram
        assert st == [1.5, 2.0] and ct == [1, 2]   # MAX of statistics, SUM of violation counts


def test_shard_ranges():
    for world in (1, 2, 4, 8):
        spans = [sdist.shard_strong(r, world, 1 << 30) for r in range(world)]
        assert spans[0][0] == 0 and sum(c for _, c in spans) == 1 << 30
        assert all(spans[i][0] + spans[i][1] == spans[i + 1][0] for i in range(world - 1))
        weak = [sdist.shard_weak(r, world, 1 << 24) for r in range(world)]
        assert all(o == r << 24 and c == 1 << 24 for r, (o, c) in enumerate(weak))
    with pytest.raises(ValueError):
        sdist.shard_weak(2, 2, 10)


def test_launch_plan_enforces_gpu_count():
    """bench.py --gpus N: re-exec under torchrun when N > 1 and no torchrun environment exists;
    refuse a torchrun job whose WORLD_SIZE differs from N (no silent 1-GPU number)."""
    assert sdist.launch_plan(1, {}) == ("run", 1)
    assert sdist.launch_plan(8, {}) == ("exec", 8)
    assert sdist.launch_plan(4, {"WORLD_SIZE": "4"}) == ("run", 4)
    assert sdist.launch_plan(1, {"WORLD_SIZE": "1"}) == ("run", 1)
    for gpus, env in ((8, {"WORLD_SIZE": "1"}), (1, {"WORLD_SIZE": "2"}), (0, {})):
        with pytest.raises(ValueError):
            sdist.launch_plan(gpus, env)
    argv = sdist.torchrun_argv("py", "/x/bench.py", 8, 29500, ["--gpus", "8", "--steps", "3"])
    assert argv[:3] == ["py", "-m", "torch.distributed.run"]
    assert "--nproc-per-node=8" in argv and "--master-addr=127.0.0.1" in argv
    assert argv[-5:] == ["/x/bench.py", "--gpus", "8", "--steps", "3"]


def test_accuracy_sample_is_rank_invariant():
    """The max_ulp_err sample: the union over ranks of each rank's local indices (shifted by its
    offset) is the same global sample for R = 1, 2, 4, 8, strong and weak layouts."""
    n = (1 << 30) + 7
    ref = sdist.sample_indices(n, 20_000, 0, n)
    assert len(ref) == 20_000 and ref[0] == 0 and ref[-1] == n - 1
    for R in (2, 4, 8):
        parts = []
        for r in range(R):
            off, cnt = sdist.shard_strong(r, R, n)
            loc = sdist.sample_indices(n, 20_000, off, cnt)
            assert ((loc >= 0) & (loc < cnt)).all()
            parts.append(loc + off)
        assert np.array_equal(np.concatenate(parts), ref)


def test_bench_reexec_argv(tmp_path):
    """bench.py --gpus 2 without torchrun execs torchrun (checked without running it: the
    planned argv is printed by a dry-run of the same helper bench.py uses)."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = ("import sys; sys.argv=['bench.py','--gpus','2']; sys.path.insert(0, %r);"
            "from paper_2510_09892_b200 import dist as d; import os;"
            "os.environ.pop('WORLD_SIZE', None); print(d.launch_plan(2))" % root)
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=60)
    assert "('exec', 2)" in out.stdout
