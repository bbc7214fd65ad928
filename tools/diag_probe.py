"""Diagnostic for the eye-frame tile probe: per-ray walk cost of the config-2 frame (stats
build of the trace kernel) -> for each probe budget B, which 8x4 tiles the probe ray (lane 12)
flags (fetches > B) against each tile's true cost (its slowest lane's iterations)."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2603_00292_b200 import accel, compile_scene, scenes  # noqa: E402
from paper_2603_00292_b200.integrators import raygen  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "sphere"
if which == "soup":
    desc, W, H = scenes.soup_description(), 3840, 2160
else:
    desc, W, H = scenes.sphere_description(), 1920, 1080
sc = compile_scene(desc)
rays = raygen(sc, W, H)
hits = torch.empty((W * H, 4), device="cuda")
st = torch.empty((W * H, 2), dtype=torch.int32, device="cuda")
accel.trace_closest(sc.tlas, rays, hits, stats=st)
torch.cuda.synchronize()
s = st.cpu().numpy().astype(np.int64)
cost = (s[:, 0] + s[:, 1]).reshape(H, W)
fetch = s[:, 1].reshape(H, W)
np.savez_compressed(f"gpurun_out/diag_probe_{which}.npz", cost=cost.astype(np.int32), fetch=fetch.astype(np.int32))
tmax = cost.reshape(H // 4, 4, W // 8, 8).max(axis=(1, 3))
probe = fetch.reshape(H // 4, 4, W // 8, 8)[:, 1, :, 4]
out = {"tiles": int(tmax.size)}
for thr in (100, 150):
    true = tmax >= thr
    out[f"true>={thr}"] = int(true.sum())
    for b in (8, 12, 16, 20, 24, 32):
        flag = probe > b
        out[f"true>={thr}_B{b}"] = {"flagged": int(flag.sum()), "caught": int((flag & true).sum())}
print(json.dumps(out))
