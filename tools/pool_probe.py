"""Does compile_scene's pool allocation block the host?  rt_scene_compile host time with the
previous scene alive (the e2e loop) vs freed first, and with a warm pool trimmed or not."""
import dataclasses
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from paper_2603_00292_b200 import _native, compile_scene, render_frame, scenes
    from paper_2603_00292_b200._native import host_pinned_copy
    from paper_2603_00292_b200.scene_io import TriangleMesh
    desc = scenes.sphere_description()
    mesh = desc.meshes["mesh"]
    pm = TriangleMesh(host_pinned_copy(np.ascontiguousarray(mesh.vertices, np.float64)),
                      host_pinned_copy(np.ascontiguousarray(mesh.faces, np.int64)))
    pdesc = dataclasses.replace(desc, meshes={"mesh": pm})
    real = _native.lib()
    acc = {}

    class T:
        def __getattr__(self, n):
            f = getattr(real, n)

            def c(*a):
                t0 = time.perf_counter()
                r = f(*a)
                acc[n] = acc.get(n, 0.0) + time.perf_counter() - t0
                return r
            return c
    for mode in ("keep", "del", "keep+render", "del+render"):
        s = compile_scene(pdesc)
        for _ in range(3):
            s = compile_scene(pdesc)
        torch.cuda.synchronize()
        acc.clear()
        _native._lib = T()
        t0 = time.perf_counter()
        for _ in range(20):
            if mode.startswith("del"):
                del s
            s = compile_scene(pdesc)
            if mode.endswith("render"):
                render_frame(s, 1920, 1080, 1, "eye")
            torch.cuda.synchronize()
        tt = (time.perf_counter() - t0) / 20
        _native._lib = real
        print(mode, f"step {tt * 1e3:.3f} ms", {k: round(v / 20 * 1e3, 3) for k, v in acc.items() if v / 20 > 2e-5})


if __name__ == "__main__" and len(sys.argv) == 1:
    main()


def profile_keep():
    """The slow host calls of the keep+render loop (torch.profiler)."""
    import torch
    from torch.profiler import ProfilerActivity, profile
    from paper_2603_00292_b200 import compile_scene, render_frame, scenes
    from paper_2603_00292_b200._native import host_pinned_copy
    from paper_2603_00292_b200.scene_io import TriangleMesh
    desc = scenes.sphere_description()
    mesh = desc.meshes["mesh"]
    pm = TriangleMesh(host_pinned_copy(np.ascontiguousarray(mesh.vertices, np.float64)),
                      host_pinned_copy(np.ascontiguousarray(mesh.faces, np.int64)))
    pdesc = dataclasses.replace(desc, meshes={"mesh": pm})
    s = compile_scene(pdesc)
    for _ in range(3):
        s = compile_scene(pdesc)
        render_frame(s, 1920, 1080, 1, "eye")
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
        for _ in range(2):
            s = compile_scene(pdesc)
            render_frame(s, 1920, 1080, 1, "eye")
        torch.cuda.synchronize()
    ev = list(prof.events())
    t0 = min(e.time_range.start for e in ev)
    for e in sorted(ev, key=lambda e: e.time_range.start):
        d = (e.time_range.end - e.time_range.start) / 1e3
        if d > 0.1 and e.name.startswith("cuda"):
            print(f"  slow {(e.time_range.start - t0) / 1e3:9.3f} ms  {d:7.3f}  {e.name}")


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "prof":
    profile_keep()


def pool_stats():
    """Default-pool reserved / used bytes around each step of the keep+render loop."""
    import torch
    from cuda.bindings import runtime as rt
    from paper_2603_00292_b200 import compile_scene, render_frame, scenes
    from paper_2603_00292_b200._native import host_pinned_copy
    from paper_2603_00292_b200.scene_io import TriangleMesh
    desc = scenes.sphere_description()
    mesh = desc.meshes["mesh"]
    pm = TriangleMesh(host_pinned_copy(np.ascontiguousarray(mesh.vertices, np.float64)),
                      host_pinned_copy(np.ascontiguousarray(mesh.faces, np.int64)))
    pdesc = dataclasses.replace(desc, meshes={"mesh": pm})
    _, pool = rt.cudaDeviceGetDefaultMemPool(0)

    def st():
        r = rt.cudaMemPoolGetAttribute(pool, rt.cudaMemPoolAttr.cudaMemPoolAttrReservedMemCurrent)[1]
        u = rt.cudaMemPoolGetAttribute(pool, rt.cudaMemPoolAttr.cudaMemPoolAttrUsedMemCurrent)[1]
        t = rt.cudaMemPoolGetAttribute(pool, rt.cudaMemPoolAttr.cudaMemPoolAttrReleaseThreshold)[1]
        return f"reserved {int(r) >> 20} MB used {int(u) >> 20} MB thr {int(t)}"
    s = compile_scene(pdesc)
    for i in range(6):
        t0 = time.perf_counter()
        s = compile_scene(pdesc)
        t1 = time.perf_counter()
        a = st()
        render_frame(s, 1920, 1080, 1, "eye")
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        print(f"step {i}: compile {1e3 * (t1 - t0):.2f} ms ({a}), render {1e3 * (t2 - t1):.2f} ms ({st()})")


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "stats":
    pool_stats()
