"""Diagnostic: distribution of per-ray walk cost (triangle tests, BVH4 node fetches) of the
config-2 eye frame (1080p, 1M sphere) and where the heaviest rays sit in the image."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2603_00292_b200 import accel, compile_scene, scenes  # noqa: E402
from paper_2603_00292_b200.integrators import raygen  # noqa: E402

W, H = 1920, 1080
sc = compile_scene(scenes.sphere_description())
rays = raygen(sc, W, H)
hits = torch.empty((W * H, 4), device="cuda")
st = torch.empty((W * H, 2), dtype=torch.int32, device="cuda")
accel.trace_closest(sc.tlas, rays, hits, stats=st)
torch.cuda.synchronize()
s = st.cpu().numpy().astype(np.int64)
tests, fetch = s[:, 0], s[:, 1]
cost = tests + fetch
out = {}
for name, v in (("tests", tests), ("fetch", fetch), ("iters", cost)):
    out[name] = {q: int(np.percentile(v, q)) for q in (50, 90, 99, 99.9, 99.99)}
    out[name]["max"] = int(v.max())
    out[name]["mean"] = float(v.mean())
for thr in (50, 100, 200, 400, 800):
    idx = np.nonzero(cost > thr)[0]
    y, x = idx // W, idx % W
    out[f"iters>{thr}"] = {"count": int(len(idx)), "rows": [int(y.min()), int(y.max())] if len(idx) else None,
                           "cols": [int(x.min()), int(x.max())] if len(idx) else None,
                           "iter_sum": int(cost[idx].sum())}
out["iter_sum_all"] = int(cost.sum())
top = np.argsort(-cost)[:12]
out["top"] = [[int(i // W), int(i % W), int(tests[i]), int(fetch[i])] for i in top]
# cost by 8x4 tile (one warp batch): the batch cost is its max lane
tc = cost.reshape(H // 4, 4, W // 8, 8).max(axis=(1, 3))
out["tile_max_iters"] = {q: int(np.percentile(tc, q)) for q in (50, 90, 99, 99.9)}
out["tile_max_iters"]["max"] = int(tc.max())
print(json.dumps(out))
