"""Eye-frame time vs scene size on the UV sphere (same camera and 1080p rays): how much of
the walk's cost is memory (the working set outgrows L1/L2) vs per-step work.  Prints per
size: triangles, ms, BVH4 node fetches and triangle tests per ray (stats build), and
ns per node fetch (frame time / (rays x fetches))."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from paper_2603_00292_b200 import accel, compile_scene, render_into, scenes
    from paper_2603_00292_b200.integrators import raygen
    W, H = 1920, 1080
    acc = torch.zeros((H * W, 4), dtype=torch.float32, device="cuda")
    out = []
    for st, sl in ((125, 250), (250, 500), (500, 1000), (1000, 2000), (1400, 2800)):
        sc = compile_scene(scenes.sphere_description(st, sl))
        rays = raygen(sc, W, H)
        hits = torch.empty((W * H, 4), dtype=torch.float32, device="cuda")
        stt = torch.empty((W * H, 2), dtype=torch.int32, device="cuda")
        accel.trace_closest(sc.tlas, rays, hits, stats=stt)
        torch.cuda.synchronize()
        nt, nn = float(stt[:, 0].double().mean()), float(stt[:, 1].double().mean())
        for _ in range(3):
            render_into(sc, acc, W, H, 1, "eye", count_rays=False)
        torch.cuda.synchronize()
        ts = []
        for _ in range(15):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            render_into(sc, acc, W, H, 1, "eye", count_rays=False)
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        ms = float(np.median(ts))
        out.append({"tris": sc.tlas.n, "ms": round(ms, 4), "node_fetches": round(nn, 2), "tri_tests": round(nt, 2),
                    "ns_per_fetch_per_ray": round(1e6 * ms / (W * H * nn), 4)})
        print(json.dumps(out[-1]), flush=True)
        del sc


if __name__ == "__main__":
    main()
