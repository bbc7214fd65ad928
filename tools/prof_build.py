"""LBVH build stage timings (device ms, CUDA events per stage) on the config-2 sphere
and the config-4 soup; optional trace timing of the config-2 eye frame.

    python tools/prof_build.py [--soup N] [--reps R] [--trace]
"""

import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--soup", type=int, default=10_000_000)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--trace", action="store_true")
    a = ap.parse_args()
    import torch
    from paper_2603_00292_b200 import compile_scene, scenes
    from paper_2603_00292_b200.integrators import render_into
    out = {}
    descs = {"sphere1M": scenes.sphere_description()}
    if a.soup:
        descs[f"soup{a.soup}"] = scenes.soup_description(a.soup)
    for name, desc in descs.items():
        sc = compile_scene(desc, "lbvh30", device=0)
        for bits in (30, 63):
            for _ in range(3):
                sc.tlas.build_profiled(bits)
            acc = {}
            tot = []
            for _ in range(a.reps):
                st = sc.tlas.build_profiled(bits)
                for k, v in st.items():
                    acc[k] = acc.get(k, 0.0) + v / a.reps
                tot.append(sum(st.values()))
            ms = [sc.tlas.build(bits, timed=True) for _ in range(a.reps)]
            out[f"{name}/{bits}"] = {"stages": {k: round(v, 4) for k, v in acc.items()},
                                     "sum_ms": round(float(np.mean(tot)), 4),
                                     "build_ms_median": round(float(np.median(ms)), 4)}
        if a.trace and name == "sphere1M":
            sc.tlas.build(30)
            W, H = 1920, 1080
            accb = torch.zeros((H * W, 4), dtype=torch.float32, device="cuda")
            for _ in range(3):
                render_into(sc, accb, W, H, 1, "eye", count_rays=False)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ts = []
            for _ in range(a.reps):
                e0.record()
                render_into(sc, accb, W, H, 1, "eye", count_rays=False)
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            out["eye1080_ms_median"] = round(float(np.median(ts)), 4)
        del sc
    if a.trace:
        from paper_2603_00292_b200 import IntegratorConfig
        cs = compile_scene(scenes.cornell_description(), "lbvh30", device=0)
        W, H = 1920, 1080
        accb = torch.zeros((H * W, 4), dtype=torch.float32, device="cuda")
        cfg = IntegratorConfig(max_depth=5)
        for kern in ("mega", "wavefront"):
            render_into(cs, accb, W, H, 2, "pt", cfg=cfg, kernel=kern, count_rays=False)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            render_into(cs, accb, W, H, 8, "pt", cfg=cfg, kernel=kern, count_rays=False)
            e1.record()
            torch.cuda.synchronize()
            out[f"pt1080x8spp_{kern}_ms"] = round(e0.elapsed_time(e1), 3)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
