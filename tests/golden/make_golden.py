"""Generate the golden fixtures in tests/golden/ by running the REFERENCE itself.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py            # all fixtures
    python tests/golden/make_golden.py spheres    # only spheres.npz
    python tests/golden/make_golden.py cli        # only cli_ppm.npz (reference CLI PPM bytes)

It imports the reference ``pathtrace`` package from /root/reference/pkg/src
(numba CPU library) and records its outputs on small, seeded inputs.  The
fixtures pin the float64 oracle (oracle/, checked bit-exactly in
tests/test_oracle_golden.py) and give the GPU tests reference answers that do
not need /root/reference at run time.
"""

import os
import sys
import tempfile

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))


def import_reference():
    os.environ.setdefault("NUMBA_CACHE_DIR", os.path.join(tempfile.gettempdir(), "numba_ref_cache"))
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import pathtrace  # noqa: F401
    return pathtrace


def ref_scene(pt, desc, quality="balanced"):
    from pathtrace.scene import compile_scene
    return compile_scene(desc, quality)


def ref_desc_from_mesh(pt, V, F, origin, right, up, color=(0.8, 0.8, 0.8)):
    from pathtrace.scene_io import SceneDescription, TriangleMesh, InstanceDecl
    from pathtrace.integrators import Material
    cam = pt.Camera(np.asarray(origin, float), np.asarray(right, float), np.asarray(up, float))
    return SceneDescription(cam, {"mesh": TriangleMesh(V, F)}, {"mesh": "<synthetic>"},
                            {"m": Material(np.array(color, float))}, [InstanceDecl("mesh", "m")], [],
                            np.zeros(3), np.zeros(3))


def primary_rays(pt, scene, W, H, seed=0, s=0, jitter=True):
    """Exactly the reference's raygen (integrators.py:345-351, camera.py:81-97), float64."""
    cam = scene.camera
    O = np.tile(cam.origin, (W * H, 1))
    D = np.empty((W * H, 3))
    for pix in range(W * H):
        xi, yi = pix % W, pix // W
        st = pt.RandomStream.for_sample(seed, pix, s)
        ju = st.uniform() if jitter else 0.0
        jv = st.uniform() if jitter else 0.0
        u, v = pt.pixel_to_uv(xi, yi, W, H, ju, jv)
        D[pix] = pt.primary_ray(cam, u, v).direction
    return O, D


def make_spheres(pt):
    """7. spheres.scn (custom-primitive sphere instances, scene.py:101-112): hits, any-hit,
    the registry error and render_frame accumulations, all from the reference."""
    from pathtrace.integrators import IntegratorConfig
    desc = pt.load_scene("/root/reference/pkg/scenes/spheres.scn")
    sc = ref_scene(pt, desc)
    out = {}
    O, D = primary_rays(pt, sc, 48, 36)
    r = pt.closest_hit_batch(sc.tlas, O, D, registry=sc.registry, with_stats=True)
    for k, val in zip(("t", "inst", "prim", "u", "v", "n", "stats"), r):
        out["p_" + k] = val
    out["O"], out["D"] = O, D
    rng = np.random.default_rng(7)
    m = 4000
    # rays from points around the spheres toward random directions (many start inside
    # or graze a sphere), plus rays aimed at sphere centers from outside
    RO = rng.uniform((-2.5, 0.01, -2.8), (2.5, 2.2, 1.2), (m, 3))
    RD = rng.normal(size=(m, 3))
    ctr = np.array([[-1.3, 0.6, 0.0], [1.3, 0.6, 0.0], [0.0, 0.9, -1.6]])
    aim = ctr[np.arange(m) % 3] + rng.normal(scale=0.5, size=(m, 3))
    RD[m // 2:] = aim[m // 2:] - RO[m // 2:]
    RD /= np.linalg.norm(RD, axis=1, keepdims=True)
    RD[m // 2:] *= rng.uniform(0.5, 2.0, (m - m // 2, 1))     # unnormalised directions too
    tmin = np.where(np.arange(m) % 7 == 0, 0.05, 0.0)
    tmax = np.where(np.arange(m) % 5 == 0, 1.5, 1e30)
    r = pt.closest_hit_batch(sc.tlas, RO, RD, tmin, tmax, registry=sc.registry, with_stats=True)
    for k, val in zip(("t", "inst", "prim", "u", "v", "n", "stats"), r):
        out["r_" + k] = val
    out["RO"], out["RD"], out["tmin"], out["tmax"] = RO, RD, tmin, tmax
    out["r_any"] = pt.any_hit_batch(sc.tlas, RO, RD, tmin, tmax, registry=sc.registry)
    # ray_mask selecting only the mesh instances would need masks; the scene uses
    # full masks, so the masked case is all misses -- keep the registry=None error
    try:
        pt.closest_hit_batch(sc.tlas, O, D)
        out["noreg_error"] = np.array("")
    except Exception as exc:                       # RegistryError
        out["noreg_error"] = np.array(f"{type(exc).__name__}: {exc}")
    meta = dict(inverses=sc.tlas.inverses, diag=np.array(sc.diagonal()), inst_material=sc.inst_material,
                root_box=sc.tlas.nodes["bounds"][0])
    out.update({"meta_" + k: v for k, v in meta.items()})
    for name, integ, w, h, spp, md in (("eye", "eye", 32, 24, 2, 8), ("pt", "pt", 24, 18, 4, 5),
                                       ("ao", "ao", 16, 12, 2, 8), ("nee", "pt-nee", 16, 12, 4, 5)):
        cfg = IntegratorConfig(max_depth=md, ao_ray_count=8)
        acc, st = pt.render_frame(sc, w, h, spp, integ, seed=0, workers=2, cfg=cfg, return_stats=True)
        out["render_" + name] = acc.data
        out["render_" + name + "_rays"] = np.array(st["rays"])
        out["render_" + name + "_args"] = np.array([w, h, spp, md])
    np.savez_compressed(os.path.join(HERE, "spheres.npz"), **out)


CLI_JOBS = (
    ("cornell_eye", "cornell", ["--width", "64", "--height", "48", "--spp", "2", "--integrator", "eye"]),
    ("cornell_pt", "cornell", ["--width", "32", "--height", "24", "--spp", "4", "--integrator", "pt",
                               "--max-depth", "5"]),
    ("cornell_ao", "cornell", ["--width", "24", "--height", "16", "--spp", "2", "--integrator", "ao",
                               "--ao-rays", "4", "--no-gamma"]),
    ("spheres_eye", "spheres", ["--width", "48", "--height", "36", "--spp", "1", "--integrator", "eye"]),
    ("spheres_nee", "spheres", ["--width", "24", "--height", "18", "--spp", "2", "--integrator", "pt-nee",
                                "--max-depth", "4", "--seed", "3"]),
)


def make_cli(pt):
    """8. the reference CLI (cli.py:45-101) end to end: PPM bytes for scene files written
    from the package's built-in descriptions (scene_io.write_scene_files)."""
    from pathtrace.cli import run
    sys.path.insert(0, ROOT)
    from paper_2603_00292_b200 import scenes
    from paper_2603_00292_b200.scene_io import write_scene_files
    out = {}
    with tempfile.TemporaryDirectory() as tmp:
        paths = {"cornell": write_scene_files(scenes.cornell_description(), os.path.join(tmp, "c")),
                 "spheres": write_scene_files(scenes.spheres_description(), os.path.join(tmp, "s"))}
        for name, scn, args in CLI_JOBS:
            ppm = os.path.join(tmp, name + ".ppm")
            rc = run(["--scene", paths[scn], "--out", ppm] + args)
            assert rc == 0, (name, rc)
            out[name] = np.frombuffer(open(ppm, "rb").read(), dtype=np.uint8)
    np.savez_compressed(os.path.join(HERE, "cli_ppm.npz"), **out)


def main():
    pt = import_reference()
    if sys.argv[1:] == ["spheres"]:
        make_spheres(pt)
        return
    if sys.argv[1:] == ["cli"]:
        make_cli(pt)
        return
    from pathtrace.accel import _build_bvh
    from pathtrace.integrators import IntegratorConfig
    sys.path.insert(0, ROOT)
    from paper_2603_00292_b200 import scenes

    out = {}
    # 1. RNG -----------------------------------------------------------------
    streams = [(0, 0, 0), (0, 1, 0), (1, 12345, 63), (2**64 - 1, 7, 3), (123456789, 2**40, 1000),
               (0, 65535, 0), (5, 2073599, 1023)]
    uni = []
    states = []
    for (sd, px, s) in streams:
        st = pt.RandomStream.for_sample(sd, px, s)
        states.append((st._state, st._inc))
        uni.append([st.uniform() for _ in range(8)])
    kat = pt.RandomStream(42, 54)
    np.savez_compressed(os.path.join(HERE, "pcg.npz"),
                        streams=np.array(streams, dtype=np.uint64), uniforms=np.array(uni),
                        states=np.array(states, dtype=np.uint64),
                        kat_u32=np.array([kat.next_u32() for _ in range(6)], dtype=np.uint64))

    # 2. Cornell box ------------------------------------------------------------
    desc = pt.load_scene("/root/reference/pkg/scenes/cornell.scn")
    sc = ref_scene(pt, desc)
    W = H = 64
    O, D = primary_rays(pt, sc, W, H)
    t, inst, prim, u, v, n, stats = pt.closest_hit_batch(sc.tlas, O, D, with_stats=True)
    rng = np.random.default_rng(1)
    m = 3000
    RO = rng.uniform(0.02, 0.98, (m, 3))
    RD = rng.normal(size=(m, 3))
    RD /= np.linalg.norm(RD, axis=1, keepdims=True)
    RD[:100, 0] = 0.0                       # exact-zero direction components
    RD[100:150, 1] = 0.0
    tmin = np.where(np.arange(m) % 7 == 0, 0.05, 0.0)
    tmax = np.where(np.arange(m) % 5 == 0, 0.5, 1e30)
    rt, ri, rp, ru, rv, rn, rs = pt.closest_hit_batch(sc.tlas, RO, RD, tmin, tmax, with_stats=True)
    rany = pt.any_hit_batch(sc.tlas, RO, RD, tmin, tmax)
    mt, mi, mp, _, _, _ = pt.closest_hit_batch(sc.tlas, RO, RD, tmin, tmax, ray_mask=0x0)
    meta = dict(inverses=sc.tlas.inverses, matrices=sc.tlas.matrices, cam=np.array([*sc.camera.origin,
                *sc.camera.right, *sc.camera.up, *sc.camera.forward, sc.camera.distortion]),
                diag=np.array(sc.diagonal()), lv0=sc.lights.v0, lv1=sc.lights.v1, lv2=sc.lights.v2,
                ln=sc.lights.normal, lemis=sc.lights.emissive, larea=sc.lights.area,
                inst_material=sc.inst_material, mat_color=sc.mat_color, mat_emissive=sc.mat_emissive,
                root_box=sc.tlas.nodes["bounds"][0])
    np.savez_compressed(os.path.join(HERE, "cornell_hits.npz"), O=O, D=D, t=t, inst=inst, prim=prim, u=u, v=v,
                        n=n, stats=stats, RO=RO, RD=RD, tmin=tmin, tmax=tmax, rt=rt, ri=ri, rp=rp, ru=ru, rv=rv,
                        rn=rn, rs=rs, rany=rany, masked_t=mt, **{"meta_" + k: v for k, v in meta.items()})

    # 3. Cornell renders (render_frame) ----------------------------------------
    renders = {}
    jobs = [("eye32", "eye", 32, 32, 2, 0, True, 8), ("eye16c", "eye", 16, 16, 1, 0, False, 8),
            ("pt24", "pt", 24, 24, 4, 0, True, 5), ("pt16s7", "pt", 16, 16, 3, 7, True, 8),
            ("ao16", "ao", 16, 16, 2, 0, True, 8), ("nee16", "pt-nee", 16, 16, 4, 0, True, 5)]
    for name, integ, w, h, spp, seed, jit, md in jobs:
        cfg = IntegratorConfig(max_depth=md, ao_ray_count=8)
        acc, st = pt.render_frame(sc, w, h, spp, integ, seed=seed, workers=2, cfg=cfg, jitter=jit,
                                  return_stats=True)
        renders[name] = acc.data
        renders[name + "_rays"] = np.array(st["rays"])
        renders[name + "_args"] = np.array([w, h, spp, seed, int(jit), md])
    np.savez_compressed(os.path.join(HERE, "cornell_render.npz"), **renders)

    # 4. SAH build arrays --------------------------------------------------------
    bv = {}
    soup = scenes.random_soup(500, seed=3)
    sph = scenes.uv_sphere(10, 20)
    for tag, mesh in (("soup", soup), ("sphere", sph)):
        tri = mesh.vertices[mesh.faces]
        lo, hi = tri.min(axis=1), tri.max(axis=1)
        bv[tag + "_lo"], bv[tag + "_hi"] = lo, hi
        for q in ("balanced", "fast"):
            nd = _build_bvh(lo, hi, q)
            for k in ("bounds", "left", "right", "count", "axis", "order"):
                bv[f"{tag}_{q}_{k}"] = nd[k]
            bv[f"{tag}_{q}_depth"] = np.array(nd["depth"])
    np.savez_compressed(os.path.join(HERE, "bvh_sah.npz"), **bv)

    # 5. sphere + soup primary hits (synthetic configs at test size) -------------
    syn = {}
    for tag, mesh, cam in (("sphere", scenes.uv_sphere(50, 100), ((0, 0, 2.5), (0.8, 0, 0), (0, 0.45, 0))),
                           ("soup", scenes.random_soup(4000, seed=0),
                            ((0.5, 0.5, 2.5), (0.6222, 0, 0), (0, 0.35, 0)))):
        d2 = ref_desc_from_mesh(pt, mesh.vertices, mesh.faces, *cam)
        s2 = ref_scene(pt, d2)
        O2, D2 = primary_rays(pt, s2, 48, 27)
        r = pt.closest_hit_batch(s2.tlas, O2, D2, with_stats=True)
        for k, val in zip(("t", "inst", "prim", "u", "v", "n", "stats"), r):
            syn[f"{tag}_{k}"] = val
        syn[f"{tag}_O"], syn[f"{tag}_D"] = O2, D2
        acc = pt.render_frame(s2, 48, 27, 1, "eye", seed=0)
        syn[f"{tag}_eye"] = acc.data
    np.savez_compressed(os.path.join(HERE, "synthetic_hits.npz"), **syn)

    # 6. scalar triangle test incl. SPEC.md:63-71 examples ---------------------
    from pathtrace.geometry import intersect_ray_triangle_batch
    k = 4000
    g = np.random.default_rng(2)
    v0, v1, v2 = (g.normal(size=(k, 3)) for _ in range(3))
    o = g.normal(size=(k, 3)) * 2
    tgt = (v0 + v1 + v2) / 3 + g.normal(size=(k, 3)) * 0.5
    d = tgt - o
    tmn = np.zeros(k)
    tmx = np.full(k, 1e30)
    o[0], d[0], v0[0], v1[0], v2[0] = (0.25, 0.25, -1), (0, 0, 1), (0, 0, 0), (1, 0, 0), (0, 1, 0)
    o[1], d[1] = (0.25, 0.25, -1), (1, 0, 0)
    res = intersect_ray_triangle_batch(o, d, tmn, tmx, v0, v1, v2)
    np.savez_compressed(os.path.join(HERE, "tri_hit.npz"), o=o, d=d, v0=v0, v1=v1, v2=v2, out=res)
    make_spheres(pt)
    make_cli(pt)
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
