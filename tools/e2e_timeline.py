"""GPU timeline of the config-2 end-to-end step (compile_scene + render_frame('eye') from
pinned float64/int64 host arrays) via torch.profiler (CUPTI): every kernel and memcpy of one
step with its start/end relative to the step's first GPU activity, and the host-side span of
each API call, to see where the step's wall time goes beyond the PCIe copies."""
import dataclasses
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from torch.profiler import ProfilerActivity, profile, record_function
    from paper_2603_00292_b200 import compile_scene, render_frame, scenes
    from paper_2603_00292_b200._native import host_pinned_copy
    from paper_2603_00292_b200.scene_io import TriangleMesh
    desc = scenes.sphere_description()
    mesh = desc.meshes["mesh"]
    pm = TriangleMesh(host_pinned_copy(np.ascontiguousarray(mesh.vertices, np.float64)),
                      host_pinned_copy(np.ascontiguousarray(mesh.faces, np.int64)))
    pdesc = dataclasses.replace(desc, meshes={"mesh": pm})
    W, H = 1920, 1080
    for _ in range(5):
        render_frame(compile_scene(pdesc, "lbvh30"), W, H, 1, "eye")
    torch.cuda.synchronize()
    def step(i):                                # the scene dies with the step (as in bench.py)
        with record_function(f"step{i}"):
            with record_function("compile_scene"):
                s2 = compile_scene(pdesc, "lbvh30")
            with record_function("render_frame"):
                render_frame(s2, W, H, 1, "eye")

    for i in range(3):
        step(i)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
        for i in range(3):
            step(i)
    ev = [e for e in prof.events()]
    steps = sorted([e for e in ev if e.name.startswith("step")], key=lambda e: e.time_range.start)
    last = steps[-1]
    t0, t1 = last.time_range.start, last.time_range.end
    print(f"host span of the step: {(t1 - t0) / 1e3:.3f} ms")
    for e in ev:
        if e.name in ("compile_scene", "render_frame") and t0 <= e.time_range.start <= t1:
            print(f"  host {e.name}: {(e.time_range.start - t0) / 1e3:.3f} .. {(e.time_range.end - t0) / 1e3:.3f} ms")
    gpu = [e for e in ev if e.device_type == torch.autograd.DeviceType.CUDA and t0 <= e.time_range.start <= t1 + 5000]
    gpu.sort(key=lambda e: e.time_range.start)
    for e in gpu:
        print(f"  gpu {(e.time_range.start - t0) / 1e3:8.3f} .. {(e.time_range.end - t0) / 1e3:8.3f} ms  "
              f"{(e.time_range.end - e.time_range.start) / 1e3:7.3f}  {e.name[:70]}")
    # API calls on the host (cudaMemcpyAsync, cudaStreamSynchronize ...) in the step
    api = [e for e in ev if e.device_type == torch.autograd.DeviceType.CPU and e.name.startswith("cuda")
           and t0 <= e.time_range.start <= t1]
    agg = {}
    for e in api:
        agg.setdefault(e.name, [0, 0.0])
        agg[e.name][0] += 1
        agg[e.name][1] += (e.time_range.end - e.time_range.start) / 1e3
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"  api {k}: {n} calls, {t:.3f} ms")
    for e in sorted(api, key=lambda e: e.time_range.start):   # the host calls that block
        d = (e.time_range.end - e.time_range.start) / 1e3
        if d > 0.02:
            print(f"  slow api {(e.time_range.start - t0) / 1e3:8.3f} .. {(e.time_range.end - t0) / 1e3:8.3f} ms  {e.name}")


if __name__ == "__main__":
    main()
