"""Breakdown of bench.py's config-2 e2e step (host buffers): refit (vertex H2D + rebuild)
and closest_hit_batch (float64 rays in, reference dtypes out), each timed alone."""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from paper_2603_00292_b200 import closest_hit_batch, compile_scene, scenes
    from paper_2603_00292_b200._native import host_pinned_copy
    desc = scenes.sphere_description()
    sc = compile_scene(desc, "lbvh30", device=0)
    tl = sc.tlas
    W, H = 1920, 1080
    rng = np.random.default_rng(0)
    cam = np.array([0, 0, 2.5])
    u = (np.arange(W * H) % W + rng.random(W * H)) / W
    v = (np.arange(W * H) // W + rng.random(W * H)) / H
    d = np.stack([(2 * u - 1) * 0.8, (1 - 2 * v) * 0.45, -np.ones_like(u)], 1)
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    O = host_pinned_copy(np.tile(cam, (W * H, 1)))
    D = host_pinned_copy(d)
    host_tris = host_pinned_copy(tl.tris)
    out = {}

    def timed(fn, reps=5):
        fn()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(reps):
            fn()
        torch.cuda.synchronize()
        return (time.perf_counter() - t0) / reps * 1e3

    out["refit_ms"] = timed(lambda: tl.refit(host_tris, 30))
    out["closest_ms"] = timed(lambda: closest_hit_batch(sc, O, D))
    out["step_ms"] = timed(lambda: (tl.refit(host_tris, 30), closest_hit_batch(sc, O, D)))
    out["mrays_s"] = W * H / out["step_ms"] / 1e3
    print(json.dumps(out))


if __name__ == "__main__":
    main()
