"""Where the config-2 end-to-end step spends its wall time: compile_scene(desc with pinned
float64/int64 arrays) and render_frame('eye') timed apart (synchronised), then a cProfile
of a few steps (host-side Python / ctypes overheads)."""
import cProfile
import dataclasses
import os
import pstats
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from paper_2603_00292_b200 import compile_scene, render_frame, scenes
    from paper_2603_00292_b200._native import host_pinned_copy
    from paper_2603_00292_b200.scene_io import TriangleMesh
    desc = scenes.sphere_description()
    mesh = desc.meshes["mesh"]
    pm = TriangleMesh(host_pinned_copy(np.ascontiguousarray(mesh.vertices, np.float64)),
                      host_pinned_copy(np.ascontiguousarray(mesh.faces, np.int64)))
    pdesc = dataclasses.replace(desc, meshes={"mesh": pm})
    W, H = 1920, 1080
    for _ in range(3):
        render_frame(compile_scene(pdesc, "lbvh30"), W, H, 1, "eye")
    torch.cuda.synchronize()
    tc, tr = [], []
    for _ in range(10):
        t0 = time.perf_counter()
        s2 = compile_scene(pdesc, "lbvh30")
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        render_frame(s2, W, H, 1, "eye")
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        tc.append(t1 - t0)
        tr.append(t2 - t1)
    print(f"compile_scene {np.median(tc) * 1e3:.3f} ms, render_frame {np.median(tr) * 1e3:.3f} ms")
    pr = cProfile.Profile()
    pr.enable()
    for _ in range(10):
        render_frame(compile_scene(pdesc, "lbvh30"), W, H, 1, "eye")
    torch.cuda.synchronize()
    pr.disable()
    pstats.Stats(pr).sort_stats("tottime").print_stats(18)


if __name__ == "__main__":
    main()
