"""Workload for compute-sanitizer (tools, not product): the TMA-staged pair kernel on 2^20 C5
queries with special rows (so the deferred-recompute queue runs), the one-query TMA kernel, the
LDG kernel, and the fused zonal pass on a small cubed sphere (ne=32, 180 latitudes), each once.
    compute-sanitizer --tool memcheck python tools/sanitize_run.py
    compute-sanitizer --tool racecheck python tools/sanitize_run.py
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2510_09892_b200 as sgi  # noqa: E402
import sgi_inputs  # noqa: E402

n = 1 << 20
a, b, z0 = sgi_inputs.generate_host(5, n)
# a few meridian / pole / degenerate rows so certificates fail and the queue is exercised
idx = np.arange(11, n, 4099)
a[:, idx] = np.array([[1.0], [0.0], [0.0]]); b[:, idx] = np.array([[0.0], [0.0], [1.0]])
z0[idx] = 0.5
da, db, dz = (torch.from_numpy(x).cuda() for x in (a, b, z0))
for mode in ("eft", "naive"):
    out = torch.empty((2, 3, n), dtype=torch.float64, device="cuda")
    cnt = torch.empty(n, dtype=torch.uint8, device="cuda")
    print(mode, sgi.dispatch_path(da, db, dz, out, cnt, mode=mode))
    sgi.intersect_arc_lat(da, db, dz, mode=mode, out_xyz=out, out_count=cnt)
    ob = torch.empty(6 * n + 1, dtype=torch.float64, device="cuda")
    o1 = ob[1:].view(2, 3, n)
    print(mode, sgi.dispatch_path(da, db, dz, o1, cnt, mode=mode))
    sgi.intersect_arc_lat(da, db, dz, mode=mode, out_xyz=o1, out_count=cnt)
    m = 100_001
    sgi.intersect_arc_lat(da[:, :m].contiguous(), db[:, :m].contiguous(), dz[:m].contiguous(),
                          mode=mode)
torch.cuda.synchronize()
va, vb = sgi_inputs.cubed_sphere_edges(32)
lat = torch.from_numpy(sgi_inputs.latitudes(180)).cuda()
r = sgi.zonal_intersect(torch.from_numpy(va).cuda(), torch.from_numpy(vb).cuda(), lat, mode="eft")
torch.cuda.synchronize()
print("zonal pairs", r["cap"])
print("sanitize workload done")
