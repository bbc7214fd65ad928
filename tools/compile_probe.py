"""Where compile_scene's time goes (1M sphere, 10M soup): mesh upload + device validation,
rt_scene_compile (flatten kernels), LBVH build, total -- wall clock with syncs, after warm-up."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2603_00292_b200 import _native, compile_scene, scenes  # noqa: E402
from paper_2603_00292_b200.scene import _DeviceMesh  # noqa: E402


def t(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return 1e3 * best


def main():
    out = {}
    for label, desc in (("1M sphere", scenes.sphere_description()), ("10M soup", scenes.soup_description())):
        m = desc.meshes["mesh"]
        V = np.ascontiguousarray(m.vertices, np.float64)
        F = np.ascontiguousarray(m.faces, np.int64)
        ctx = _native.Context.get(0)
        r = {"upload_validate_ms": t(lambda: _DeviceMesh(ctx, V, F))}
        sc = compile_scene(desc)
        r["build_ms"] = t(lambda: sc.tlas.build(30))
        r["compile_scene_ms"] = t(lambda: compile_scene(desc))
        pv = _native.host_pinned_copy(V)
        pf = _native.host_pinned_copy(F)
        r["upload_validate_pinned_ms"] = t(lambda: _DeviceMesh(ctx, pv, pf))
        out[label] = r
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
