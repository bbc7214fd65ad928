"""The reference itself (pathtrace, numba, installed under baseline/_ref) timed on this host's
cores -- the round-2 record of the real CPU reference next to the float64 C port that
bench.py's --impl reference arm runs (the port cannot be beaten by a JIT warm-up, the
reference can: so both are recorded).  Run on the GPU box (same image: numba 0.65):

    python tools/ref_numba_bench.py > profiles/r2_reference_numba.json

config 2: compile_scene(sphere, "balanced" = binned SAH, and "fast") + render_frame('eye')
1920x1080 with os.cpu_count() workers; config 3: cornell.scn render_frame('pt', max_depth=5)
1920x1080 at 1 spp (the first sample of the 64-spp run).  One untimed warm-up call of each
kernel first (numba JIT).  Rays are counted by the reference (return_stats=True).
"""
import json
import os
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")
sys.path.insert(0, REF)
sys.path.insert(1, ROOT)
os.environ.setdefault("NUMBA_CACHE_DIR", os.path.join(tempfile.gettempdir(), "numba_ref_cache"))

import numpy as np  # noqa: E402
import pathtrace  # noqa: E402
from pathtrace import integrators, scene, scene_io  # noqa: E402


def ref_sphere_desc():
    """The config-2 scene through the reference's own dataclasses."""
    from paper_2603_00292_b200 import scenes
    mine = scenes.sphere_description()
    m = mine.meshes["mesh"]
    cam = pathtrace.camera.Camera(mine.camera.origin, mine.camera.right, mine.camera.up)
    mats = {k: integrators.Material(v.color, v.emissive) for k, v in mine.materials.items()}
    insts = [scene_io.InstanceDecl(d.mesh, d.material) for d in mine.instances]
    return scene_io.SceneDescription(cam, {"mesh": scene_io.TriangleMesh(m.vertices, m.faces)}, {"mesh": "mesh.obj"},
                                     mats, insts, [], np.asarray(mine.sky), np.asarray(mine.background))


def main():
    cores = os.cpu_count() or 1
    out = {"reference": "pathtrace 0.1.0 (/root/reference/pkg) installed with pip --target baseline/_ref",
           "numba": __import__("numba").__version__, "host_cores": cores}
    cfg5 = integrators.IntegratorConfig(max_depth=5)
    # JIT warm-up on a tiny scene
    corn = scene_io.load_scene(os.path.join(REF, "scenes", "cornell.scn"))
    sc = scene.compile_scene(corn)
    integrators.render_frame(sc, 16, 16, 1, "eye", workers=cores)
    integrators.render_frame(sc, 16, 16, 1, "pt", workers=cores, cfg=cfg5)
    # config 3 prefix: 1 spp of the 1080p path-traced frame
    t0 = time.perf_counter()
    _, st = integrators.render_frame(sc, 1920, 1080, 1, "pt", seed=0, workers=cores, cfg=cfg5, return_stats=True)
    dt = time.perf_counter() - t0
    out["config3_pt_1spp"] = {"rays": int(st["rays"]), "s": dt, "mrays_s": st["rays"] / dt / 1e6, "workers": cores}
    # config 2: SAH compile (fast and balanced) + the 1080p eye frame
    desc = ref_sphere_desc()
    for q in ("fast", "balanced"):
        t0 = time.perf_counter()
        s2 = scene.compile_scene(desc, q)
        tb = time.perf_counter() - t0
        t1 = time.perf_counter()
        _, st = integrators.render_frame(s2, 1920, 1080, 1, "eye", seed=0, workers=cores, return_stats=True)
        tr = time.perf_counter() - t1
        out[f"config2_{q}"] = {"compile_s": tb, "render_s": tr, "rays": int(st["rays"]),
                               "render_mrays_s": st["rays"] / tr / 1e6,
                               "step_mrays_s": st["rays"] / (tb + tr) / 1e6, "workers": cores}
        print(json.dumps(out), file=sys.stderr, flush=True)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
