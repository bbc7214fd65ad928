"""Per-tile phases of the last 10-bit onesweep pass of a config-2 (1M) build (diagnostic build:
tools/variants.sh sorttl "-DRT_SORT_TL=1"; RT_B200_LIB=variants/sorttl/librt_b200.so):
start -> tile known -> ranked -> look-back done -> scattered, in us from the first tile's
start, as percentiles over the tiles."""
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from paper_2603_00292_b200 import _native, compile_scene, scenes
    L = _native.lib()
    L.rt_debug_sort_timeline.argtypes = [ctypes.c_void_p, ctypes.c_int32]
    for name, desc in (("sphere1M", scenes.sphere_description()), ("soup10M", scenes.soup_description())):
        sc = compile_scene(desc)
        nt = min(4096, -(-sc.tlas.n // 7168))
        rows = []
        for _ in range(5):
            sc.tlas.build(30)
            torch.cuda.synchronize()
            buf = np.zeros((nt, 5), np.uint64)
            _native.check(L.rt_debug_sort_timeline(buf.ctypes.data_as(ctypes.c_void_p), nt))
            rows.append(buf.astype(np.int64))
        b = rows[-1]
        t0 = b[:, 0].min()
        rel = (b - t0) / 1e3
        ph = np.diff(b, axis=1) / 1e3
        print(f"{name}: {nt} tiles, pass span {rel[:, 4].max():.2f} us")
        for k, lab in enumerate(["launch->tile", "load+rank", "look-back(+scan)", "scatter"]):
            q = np.percentile(ph[:, k], [0, 50, 90, 100])
            print(f"  {lab:18s} min {q[0]:6.2f}  med {q[1]:6.2f}  p90 {q[2]:6.2f}  max {q[3]:6.2f} us")
        q = np.percentile(rel[:, 0], [0, 50, 100])
        print(f"  tile start offsets: min {q[0]:.2f} med {q[1]:.2f} max {q[2]:.2f} us")
        order = np.argsort(b[:, 0])
        print("  first/last tiles by start: look-back us", np.round(ph[order[:4], 2], 2), np.round(ph[order[-4:], 2], 2))


if __name__ == "__main__":
    main()
