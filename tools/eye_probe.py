"""Eye frames under the tile probe (render.cu tile_probe_kernel / tile_order_kernel):
device time and a hash of the accumulation buffer for the node-fetch budget in
RT_PROBE_BUDGET (read once per process by librt; 0 = no probe, row-major tiles).
Frames rendered with different budgets must hash identically.

    RT_PROBE_BUDGET=32 python tools/eye_probe.py [--soup] [--reps R]
"""
import argparse
import hashlib
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=15)
    ap.add_argument("--soup", action="store_true")
    ap.add_argument("--bands", type=int, default=1, help="render rank 0's share of an N-way tile-band split")
    a = ap.parse_args()
    import torch
    from paper_2603_00292_b200 import compile_scene, render_into, scenes
    out = {"budget": os.environ.get("RT_PROBE_BUDGET", "default"), "lib": os.environ.get("RT_B200_LIB", "default")}
    cases = [("sphere1080", scenes.sphere_description(), 1920, 1080)]
    if a.soup:
        cases.append(("soup4k", scenes.soup_description(), 3840, 2160))
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for name, desc, W, H in cases:
        sc = compile_scene(desc)
        acc = torch.zeros((H * W, 4), dtype=torch.float32, device="cuda")
        bands = (a.bands, 0) if a.bands > 1 else None
        render_into(sc, acc, W, H, 1, "eye", count_rays=False, bands=bands)
        torch.cuda.synchronize()
        out[f"{name}_sha"] = hashlib.sha1(acc.cpu().numpy().tobytes()).hexdigest()[:16]
        ts = []
        for k in range(a.reps):
            flush.fill_(k & 0xFF)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            render_into(sc, acc, W, H, 1, "eye", count_rays=False, bands=bands)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        out[f"{name}_ms"] = round(float(np.median(ts)), 4)
        del sc, acc
    print(json.dumps(out))


if __name__ == "__main__":
    main()
