"""Repeatability stress of the asynchronous kernels (tools, not product; the pool runs no
compute-sanitizer, so races would show as run-to-run differences):
    python tools/stress_repeat.py [zonal_passes] [eft_passes]
  * the fused zonal pass (ticketed tiles, decoupled look-back, early bulk copies, parked
    results) on the full C4 workload, every pass compared bit for bit with the first;
  * the EFT TMA pair kernel (mbarrier ring, acq_rel stage release, warp fallback queue) on C5
    2^26 and C3 2^24 (ill-conditioned: many queued recomputations), every pass compared bit for
    bit with the first.
Prints one JSON line per workload: passes, passes that differed, differing elements."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import sgi_inputs
    import paper_2510_09892_b200 as sgi
    nz = int(sys.argv[1]) if len(sys.argv) > 1 else 500
    ne_ = int(sys.argv[2]) if len(sys.argv) > 2 else 200

    va, vb = sgi_inputs.cubed_sphere_edges(1024)
    lat = sgi_inputs.latitudes(1800)
    dva, dvb = torch.from_numpy(va).cuda(), torch.from_numpy(vb).cuda()
    dl = torch.from_numpy(lat).cuda()
    first = sgi.zonal_intersect(dva, dvb, dl, mode="eft")
    torch.cuda.synchronize()
    ref = {k: v.clone() for k, v in first.items() if torch.is_tensor(v)}
    cap = int(ref["total"].item())
    bad = bad_el = 0
    for _ in range(nz):
        out = sgi.zonal_intersect(dva, dvb, dl, mode="eft", cap=cap)
        diff = 0
        for k, v in ref.items():
            a, b = out[k], v
            if a.dtype == torch.float64:
                a, b = a.view(torch.int64), b.view(torch.int64)
            diff += int((a != b).sum().item())
        bad += diff > 0
        bad_el += diff
    print(json.dumps({"workload": "zonal C4 ne=1024 x 1800", "passes": nz, "passes_differing": bad,
                      "elements_differing": bad_el, "pairs": int(ref["total"].item())}), flush=True)

    for cfg, n in ((5, 1 << 26), (3, 1 << 24)):
        a = torch.empty((3, n), dtype=torch.float64, device="cuda")
        b = torch.empty_like(a)
        z0 = torch.empty(n, dtype=torch.float64, device="cuda")
        sgi_inputs.generate_device(cfg, n, a, b, z0, seed=cfg)
        out = torch.empty((2, 3, n), dtype=torch.float64, device="cuda")
        cnt = torch.empty(n, dtype=torch.uint8, device="cuda")
        sgi.intersect_arc_lat(a, b, z0, mode="eft", out_xyz=out, out_count=cnt)
        torch.cuda.synchronize()
        r_out, r_cnt = out.view(torch.int64).clone(), cnt.clone()
        path = sgi.dispatch_path(a, b, z0, out, cnt, mode="eft")
        bad = bad_el = 0
        for _ in range(ne_):
            out.fill_(0.0)
            cnt.fill_(7)
            sgi.intersect_arc_lat(a, b, z0, mode="eft", out_xyz=out, out_count=cnt)
            diff = int((out.view(torch.int64) != r_out).sum().item()) + int((cnt != r_cnt).sum().item())
            bad += diff > 0
            bad_el += diff
        print(json.dumps({"workload": f"C{cfg} 2^{n.bit_length() - 1} eft", "kernel": path,
                          "passes": ne_, "passes_differing": bad, "elements_differing": bad_el}),
              flush=True)


if __name__ == "__main__":
    main()
