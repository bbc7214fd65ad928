"""Minimal driver for ncu: config-2 eye frame (default) or config-3 PT on Cornell.

    python tools/drive_render.py [eye|pt|ptwf|soup] [reps]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2603_00292_b200 import IntegratorConfig, compile_scene, render_into, scenes  # noqa: E402

mode = sys.argv[1] if len(sys.argv) > 1 else "eye"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
kernel = "mega"
if mode in ("pt", "ptwf"):
    sc = compile_scene(scenes.cornell_description())
    W, H, spp, integ = 1920, 1080, 1, "pt"
    kernel = "wavefront" if mode == "ptwf" else "mega"
elif mode == "soup":
    sc = compile_scene(scenes.soup_description())
    W, H, spp, integ = 3840, 2160, 1, "eye"
else:
    sc = compile_scene(scenes.sphere_description())
    W, H, spp, integ = 1920, 1080, 1, "eye"
acc = torch.zeros((W * H, 4), dtype=torch.float32, device="cuda")
for _ in range(reps):
    render_into(sc, acc, W, H, spp, integ, cfg=IntegratorConfig(max_depth=5), count_rays=False, kernel=kernel)
torch.cuda.synchronize()
