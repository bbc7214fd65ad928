"""Trace / render timings for kernel variants (device ms, CUDA events, median of reps):
1080p eye frame on the 1M sphere (config 2's trace), Cornell 1080p x 8 spp path tracing
(mega + wavefront), optionally the 4K eye frame on the 10M soup.

    RT_B200_LIB=variants/X/librt_b200.so python tools/prof_trace.py [--soup] [--reps R]
"""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def timed(fn, reps):
    import torch
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return round(float(np.median(ts)), 4)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=15)
    ap.add_argument("--soup", action="store_true")
    ap.add_argument("--no-wf", action="store_true")
    a = ap.parse_args()
    import torch
    from paper_2603_00292_b200 import IntegratorConfig, compile_scene, render_into, scenes
    out = {"lib": os.environ.get("RT_B200_LIB", "default")}
    W, H = 1920, 1080
    acc = torch.zeros((H * W, 4), dtype=torch.float32, device="cuda")
    sc = compile_scene(scenes.sphere_description())
    out["eye1080_sphere_ms"] = timed(lambda: render_into(sc, acc, W, H, 1, "eye", count_rays=False), a.reps)

    sc.tlas.build(63)
    out["eye1080_sphere_lbvh63_ms"] = timed(lambda: render_into(sc, acc, W, H, 1, "eye", count_rays=False), a.reps)
    del sc
    cs = compile_scene(scenes.cornell_description())
    cfg = IntegratorConfig(max_depth=5)
    for kern in (("mega",) if a.no_wf else ("mega", "wavefront")):
        out[f"pt1080x8_{kern}_ms"] = timed(lambda: render_into(cs, acc, W, H, 8, "pt", cfg=cfg, kernel=kern,
                                                               count_rays=False), max(3, a.reps // 3))
    if a.soup:
        W4, H4 = 3840, 2160
        acc4 = torch.zeros((H4 * W4, 4), dtype=torch.float32, device="cuda")
        ss = compile_scene(scenes.soup_description())
        out["eye4k_soup_ms"] = timed(lambda: render_into(ss, acc4, W4, H4, 1, "eye", count_rays=False), a.reps)

        ss.tlas.build(63)
        out["eye4k_soup_lbvh63_ms"] = timed(lambda: render_into(ss, acc4, W4, H4, 1, "eye", count_rays=False), a.reps)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
