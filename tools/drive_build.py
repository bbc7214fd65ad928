"""Minimal driver for ncu: compile the config-2 sphere (one build) and rebuild it R times."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_00292_b200 import compile_scene, scenes  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 2
bits = int(sys.argv[2]) if len(sys.argv) > 2 else 30
desc = scenes.soup_description() if len(sys.argv) > 3 and sys.argv[3] == "soup" else scenes.sphere_description()
sc = compile_scene(desc, "lbvh30", device=0)
for _ in range(reps):
    sc.tlas.build(bits)
sc.tlas.ctx.sync()
