"""Diagnostic: trace kernel vs eye megakernel on one scene (timings + per-ray stats)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2603_00292_b200 import accel, compile_scene, render_into, scenes  # noqa: E402
from paper_2603_00292_b200.integrators import raygen  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "soup"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 10_000_000
desc = scenes.soup_description(n) if which == "soup" else scenes.sphere_description()
W, H = (3840, 2160) if which == "soup" else (1920, 1080)
sc = compile_scene(desc)
print("height", sc.tlas.info())
rays = raygen(sc, W, H)
hits = torch.empty((W * H, 4), device="cuda")
st = torch.empty((W * H, 2), dtype=torch.int32, device="cuda")
for k in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    accel.trace_closest(sc.tlas, rays, hits, stats=st if k == 0 else None)
    torch.cuda.synchronize()
    print("trace_closest", "stats" if k == 0 else "", f"{(time.perf_counter() - t0) * 1e3:.2f} ms")
s = st.double()
print("tests mean/max", float(s[:, 0].mean()), int(s[:, 0].max()), "fetch mean/max", float(s[:, 1].mean()),
      int(s[:, 1].max()))
acc = torch.zeros((W * H, 4), device="cuda")
for k in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    render_into(sc, acc, W, H, 1, "eye", 0, None, True, "mega", count_rays=False)
    torch.cuda.synchronize()
    print("megakernel eye", f"{(time.perf_counter() - t0) * 1e3:.2f} ms")
for k in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    render_into(sc, acc, W, H, 1, "eye", 0, None, True, "wavefront", count_rays=False)
    torch.cuda.synchronize()
    print("wavefront eye", f"{(time.perf_counter() - t0) * 1e3:.2f} ms")
big = torch.nonzero(st[:, 1] > 1000).flatten()[:10].cpu().numpy()
print("rays with >1000 fetches:", int((st[:, 1] > 1000).sum()), big, rays[big].cpu().numpy() if len(big) else "")
