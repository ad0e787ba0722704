"""End-to-end (host buffers) throughput vs chunk size of sgi_intersect_arc_lat_host (tools).
    python tools/e2e_sweep.py        # on the GPU: C2, 2^24 queries, pinned host buffers"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2510_09892_b200 as sgi  # noqa: E402
if len(sys.argv) > 1:                       # time an alternative build of libsgi.so
    import paper_2510_09892_b200._build as _b
    _b.LIB_PATH = sys.argv[1]
    sgi.LIB_PATH = sys.argv[1]
import sgi_inputs  # noqa: E402

n = 1 << 24
a = torch.empty((3, n), dtype=torch.float64, device="cuda")
b = torch.empty_like(a)
z0 = torch.empty(n, dtype=torch.float64, device="cuda")
sgi_inputs.generate_device(2, n, a, b, z0)
ha, hb, hz = (t.cpu().pin_memory() for t in (a, b, z0))
hout = torch.empty((2, 3, n), dtype=torch.float64).pin_memory()
hcnt = torch.empty(n, dtype=torch.uint8).pin_memory()
for chunk in (1 << 21, 1 << 20, 1 << 19, 1 << 18, 1 << 17):
    work = torch.empty(sgi.host_workspace_bytes(chunk), dtype=torch.uint8, device="cuda")
    for mode in ("eft",):
        sgi.intersect_arc_lat_host(ha, hb, hz, mode=mode, out_xyz=hout, out_count=hcnt, work=work)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            sgi.intersect_arc_lat_host(ha, hb, hz, mode=mode, out_xyz=hout, out_count=hcnt, work=work)
        e1.record()
        torch.cuda.synchronize()
        s = e0.elapsed_time(e1) / 3 * 1e-3
        print(f"chunk {chunk:>8d} ({(n + chunk - 1) // chunk:3d} chunks) {mode}: {n / s / 1e9:.3f} G/s, "
              f"{n * 105 / s / 1e9:.1f} GB/s over PCIe", flush=True)
