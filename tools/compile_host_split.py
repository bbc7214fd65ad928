"""Host-side split of compile_scene (config-2 sphere, pinned float64/int64 arrays): time spent
inside each librt_b200 entry point vs in Python around them, per call, after warm-up."""
import dataclasses
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


class _Timed:
    def __init__(self, lib, acc):
        self._lib, self._acc = lib, acc

    def __getattr__(self, name):
        fn = getattr(self._lib, name)
        if not callable(fn):
            return fn
        acc = self._acc

        def call(*a):
            t0 = time.perf_counter()
            r = fn(*a)
            acc[name] = acc.get(name, 0.0) + time.perf_counter() - t0
            return r
        return call


def main():
    import torch
    from paper_2603_00292_b200 import _native, compile_scene, scenes
    from paper_2603_00292_b200._native import host_pinned_copy
    from paper_2603_00292_b200.scene_io import TriangleMesh
    desc = scenes.sphere_description()
    mesh = desc.meshes["mesh"]
    pm = TriangleMesh(host_pinned_copy(np.ascontiguousarray(mesh.vertices, np.float64)),
                      host_pinned_copy(np.ascontiguousarray(mesh.faces, np.int64)))
    pdesc = dataclasses.replace(desc, meshes={"mesh": pm})
    for _ in range(5):
        compile_scene(pdesc, "lbvh30")
    torch.cuda.synchronize()
    acc = {}
    real = _native.lib()
    _native._lib = _Timed(real, acc)
    n = 20
    t0 = time.perf_counter()
    for _ in range(n):
        compile_scene(pdesc, "lbvh30")
        torch.cuda.synchronize()
    total = (time.perf_counter() - t0) / n
    _native._lib = real
    inside = sum(acc.values()) / n
    print(f"compile_scene {total * 1e3:.3f} ms per call: {inside * 1e3:.3f} ms in librt, "
          f"{(total - inside) * 1e3:.3f} ms in Python / torch")
    for k, v in sorted(acc.items(), key=lambda x: -x[1]):
        print(f"  {k}: {v / n * 1e3:.3f} ms")


if __name__ == "__main__":
    main()
