"""Small end-to-end workload for compute-sanitizer (memcheck / racecheck / synccheck):
the device compile (upload + validation, the flatten kernel, a staged pageable upload),
refit_mesh with its bounds reduction, LBVH builds and in-place rebuilds (30/63-bit,
spheres), closest/any hit, all integrators, wavefront, device resolve, the render replica,
the band pack/unpack, two-level with a refresh + render, the RNG stream hook."""
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
# device compile of a mesh whose faces (47 MB) take the staged pageable upload, + refit_mesh
big = scenes.sphere_description(700, 1400)
sc = compile_scene(big)
V = big.meshes["mesh"].vertices * 1.01
sc.refit_mesh("mesh", V)
sc.diagonal()                                         # the re-reduced bounds
render_frame(sc, 32, 16, 1, "eye")
# replica + band pack / unpack
import ctypes  # noqa: E402
from paper_2603_00292_b200 import _native, distributed  # noqa: E402
cs = compile_scene(scenes.cornell_description())
rep = cs.tlas.clone(0)
acc = torch.zeros((40 * 30, 4), dtype=torch.float32, device="cuda")
comp = torch.zeros_like(acc)
for g in range(3):
    render_into(cs, acc, 40, 30, 1, "pt", 0, IntegratorConfig(max_depth=3), bands=distributed.band_split(g, 3))
    for unpack in (0, 1):
        _native.check(_native.lib().rt_bands_copy(cs.tlas.ctx.handle, _native.ptr(acc), _native.ptr(comp), 40, 30,
                                                  g, 3, unpack, None))
out = np.zeros(8, np.uint32)
_native.check(_native.lib().rt_stream_draws(cs.tlas.ctx.handle, 1, 2, 3, 8, out.ctypes.data_as(ctypes.c_void_p)))
# two-level: refit + refresh, then a render through the re-flattened copy
two = compile_scene(desc, two_level=True)
cube = names.index("cube")
two.tlas.blases[cube].refit(vertices=desc.meshes["cube"].vertices * 1.1)
two.tlas.refresh_instance_bounds()
render_frame(two, 24, 16, 2, "pt", cfg=IntegratorConfig(max_depth=3))
# tile-probe scheduling of eye frames: queue + claims (budget 24), near-everything heavy with
# the cap's early stop (budget 2), probe off
sph = compile_scene(scenes.sphere_description(200, 400))
for b in (24, 2, 0):
    _native.check(_native.lib().rt_set_probe_budget(b, None))
    acc = torch.zeros((128 * 96, 4), dtype=torch.float32, device="cuda")
    render_into(sph, acc, 128, 96, 1, "eye", count_rays=False)
    render_into(sph, acc, 128, 96, 2, "eye", count_rays=False, bands=(2, 1))
_native.check(_native.lib().rt_set_probe_budget(24, None))
torch.cuda.synchronize()
# meshes failing their (asynchronous) validation: the compile and the build are queued behind
# it, and the compile kernel must write nothing for them (out-of-range faces, non-finite rows)
import dataclasses  # noqa: E402
from paper_2603_00292_b200 import BuildError  # noqa: E402
from paper_2603_00292_b200.scene_io import TriangleMesh  # noqa: E402
Vb = rng.normal(size=(300, 3))
for bad_F, bad_V in ((np.arange(300).reshape(-1, 3) * 1000, Vb), (np.arange(300).reshape(-1, 3), np.where(Vb > 2, np.nan, Vb))):
    d0 = scenes.single_mesh_description(TriangleMesh(bad_V, bad_F), (0, 0, 3), (1, 0, 0), (0, 1, 0))
    try:
        compile_scene(d0)
        raise SystemExit("expected a BuildError")
    except BuildError:
        pass
good = compile_scene(scenes.single_mesh_description(TriangleMesh(Vb, np.arange(300).reshape(-1, 3)), (0, 0, 3),
                                                    (1, 0, 0), (0, 1, 0)))
render_frame(good, 24, 16, 1, "eye")
# eye frames of one scene and geometry in a row: probe, heavy-queue replays, a re-probe; and
# a uniformly costly soup (probe stop, then row-major frames under the hint)
sph = compile_scene(scenes.sphere_description(120, 240))
acc = torch.zeros((96 * 64, 4), dtype=torch.float32, device="cuda")
for _ in range(10):
    render_into(sph, acc, 96, 64, 1, "eye", count_rays=False)
soup = compile_scene(scenes.soup_description(200000))
acc = torch.zeros((640 * 480, 4), dtype=torch.float32, device="cuda")
for _ in range(3):
    render_into(soup, acc, 640, 480, 1, "eye", count_rays=False)
print("sanitize driver ok")
