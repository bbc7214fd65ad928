"""Small end-to-end workload for compute-sanitizer (memcheck / racecheck / synccheck):
LBVH builds and in-place rebuilds (30/63-bit, spheres), closest/any hit, all integrators,
wavefront, device resolve, two-level."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2603_00292_b200 import (Blas, Instance, IntegratorConfig, any_hit_batch, build_tlas,  # noqa: E402
                                   closest_hit_batch, compile_scene, render_frame, scenes)
from paper_2603_00292_b200.integrators import render_into, resolve_device  # noqa: E402
import torch  # noqa: E402

rng = np.random.default_rng(0)
O = rng.uniform(-1, 1, (3000, 3))
D = rng.normal(size=(3000, 3))
for desc, q in ((scenes.sphere_description(40, 80), "lbvh30"), (scenes.soup_description(20000), "lbvh63"),
                (scenes.cornell_description(), "lbvh30"), (scenes.spheres_description(), "lbvh30")):
    sc = compile_scene(desc, q)
    closest_hit_batch(sc, O, D, registry=sc.registry, with_stats=True)
    any_hit_batch(sc, O, D, registry=sc.registry)
    cfg = IntegratorConfig(max_depth=4, ao_ray_count=4)
    for integ in ("eye", "pt", "ao", "pt-nee"):
        render_frame(sc, 24, 16, 2, integ, cfg=cfg)
    render_frame(sc, 24, 16, 2, "pt", cfg=cfg, kernel="wavefront")
    acc = torch.zeros((24 * 16, 4), dtype=torch.float32, device="cuda")
    render_into(sc, acc, 24, 16, 2, "pt", 0, cfg)
    resolve_device(sc, acc, 24, 16)
    sc.tlas.refit(sc.tlas.tris)                      # rebuild in place (slot records of the last build)
desc = scenes.cornell_description()
names = list(desc.meshes)
bl = [Blas.from_mesh(desc.meshes[k].vertices, desc.meshes[k].faces) for k in names]
tl = build_tlas([Instance(names.index(d.mesh), d.frame) for d in desc.instances], bl)
closest_hit_batch(tl, O * 0.5 + 0.5, D, with_stats=True)
any_hit_batch(tl, O * 0.5 + 0.5, D)
print("sanitize driver ok")
