"""Two-level Blas / Instance / Tlas on the GPU (accel.py:211-283, 339-346, 439-549) vs the
reference's outputs (tests/golden) and the float64 two-level oracle.

Local-space rays, the reference tie rule and float64 normals (BLAS local normal
through the instance inverse transpose, accel.py:843-847) -- so normals of
agreeing triangle hits are bit-identical to the reference's.
"""

import numpy as np
import pytest

from paper_2603_00292_b200 import (Blas, Instance, RegistryError, SrtFrame, Tlas, any_hit_batch, build_tlas,
                                   closest_hit_batch, make_sphere_registry, scenes, sphere_aabbs)
from paper_2603_00292_b200.accel import SPHERE_GEOM_TYPE
from paper_2603_00292_b200.frames import FULL_MASK
from rt_helpers import golden

pytestmark = pytest.mark.gpu

T_REL = 1e-5


def tlas_from_description(desc, masks=None):
    names = list(desc.meshes)
    blases = [Blas.from_mesh(desc.meshes[k].vertices, desc.meshes[k].faces) for k in names]
    insts = [Instance(names.index(d.mesh), d.frame, d.mask if masks is None else masks[i])
             for i, d in enumerate(desc.instances)]
    reg = None
    if desc.spheres:
        rows = np.array([[*s.center, s.radius] for s in desc.spheres])
        reg = make_sphere_registry(rows)
        for k, s in enumerate(desc.spheres):
            blases.append(Blas.from_aabbs(sphere_aabbs(rows[k:k + 1]), SPHERE_GEOM_TYPE, data_offset=k))
            insts.append(Instance(len(blases) - 1, s.frame, s.mask))
    return build_tlas(insts, blases), blases, insts, reg


def _agree(res, ref, t_abs=0.0, outliers=0.0):
    t, inst, prim, u, v, n = res[:6]
    rt, ri, rp, ru, rv, rn = ref[:6]
    same = (inst == ri) & (prim == rp)
    both = same & (ri >= 0)
    rel = np.maximum(np.abs(t[both] - rt[both]) - t_abs, 0) / np.abs(rt[both])
    assert np.mean(rel > T_REL) <= outliers, rel.max()
    assert np.all(t[inst < 0] == -1.0)
    return same, both


def _only_ties(got, ref):
    """Every (inst, prim) disagreement is an exact geometric tie (cube bottoms lie flush
    with the floor at y = 0; float64 local-space and fp32 rounding break it differently)."""
    t, inst, prim = got[:3]
    rt, ri, rp = ref[:3]
    diff = (inst != ri) | (prim != rp)
    ties = diff & (inst >= 0) & (ri >= 0) & (np.abs(t - rt) <= 1e-6 * np.abs(rt))
    assert np.array_equal(diff, ties), np.nonzero(diff & ~ties)[0][:8]


def test_cornell_two_level_vs_reference(native):
    g = golden("cornell_hits")
    tl, *_ = tlas_from_description(scenes.cornell_description())
    res = closest_hit_batch(tl, g["O"], g["D"], with_stats=True)
    same, both = _agree(res, tuple(g[k] for k in ("t", "inst", "prim", "u", "v", "n")))
    assert same.all()
    # triangle normals: the reference's float64 arithmetic, bit for bit
    assert np.array_equal(res[5][both], g["n"][both])
    # (t, u, v): recomputed by the host query with the reference's float64 arithmetic (local
    # ray from the float64 inverse, _tri_hit on the float64 local vertices): bit for bit too
    exact = (res[0][both] == g["t"][both]) & (res[3][both] == g["u"][both]) & (res[4][both] == g["v"][both])
    assert exact.mean() >= 0.9999, exact.mean()
    assert np.all(res[6][:, 0] >= 1) and np.all(res[6][:, 1] >= 1)
    # random rays from inside the box: all disagreements are exact cube-bottom / floor ties
    rt, ri, rp = g["rt"], g["ri"], g["rp"]
    t, inst, prim = closest_hit_batch(tl, g["RO"], g["RD"], g["tmin"], g["tmax"])[:3]
    diff = (inst != ri) | (prim != rp)
    ties = diff & (inst >= 0) & (ri >= 0) & (np.abs(t - rt) <= 1e-6 * np.abs(rt))
    assert np.array_equal(diff, ties)
    assert np.mean(any_hit_batch(tl, g["RO"], g["RD"], g["tmin"], g["tmax"]) == g["rany"]) >= 0.9999
    m = closest_hit_batch(tl, g["RO"], g["RD"], g["tmin"], g["tmax"], ray_mask=0)
    assert np.all(m[1] == -1)


def test_spheres_two_level_vs_reference(native):
    g = golden("spheres")
    tl, blases, insts, reg = tlas_from_description(scenes.spheres_description())
    assert tl.custom_geom_types() == [SPHERE_GEOM_TYPE]
    res = closest_hit_batch(tl, g["O"], g["D"], registry=reg)
    same, both = _agree(res, tuple(g["p_" + k] for k in ("t", "inst", "prim", "u", "v", "n")))
    assert same.all()
    assert np.allclose(res[5][both], g["p_n"][both], atol=1e-6)
    res = closest_hit_batch(tl, g["RO"], g["RD"], g["tmin"], g["tmax"], registry=reg)
    same, both = _agree(res, tuple(g["r_" + k] for k in ("t", "inst", "prim", "u", "v", "n")),
                        t_abs=8 * 2.0 ** -23, outliers=1e-3)
    assert same.mean() >= 0.9999
    assert np.mean(any_hit_batch(tl, g["RO"], g["RD"], g["tmin"], g["tmax"], registry=reg) == g["r_any"]) >= 0.9999
    with pytest.raises(RegistryError, match="geometry type 0 and ray type 0"):
        closest_hit_batch(tl, g["O"], g["D"])


def test_masks_refit_refresh_vs_oracle(native, oracle_mod):
    desc = scenes.cornell_description()
    masks = [0x1, 0x2, 0x4, 0x8, 0x3, 0xF0]
    tl, blases, insts, _ = tlas_from_description(desc, masks)
    names = list(desc.meshes)

    def oracle_for(meshes, frames):
        inst = [(names.index(d.mesh), 0, f.scale, f.rotation_axis, f.rotation_angle, f.translation, masks[i])
                for i, (d, f) in enumerate(zip(desc.instances, frames))]
        return oracle_mod.OracleScene(meshes, inst, [[0.5] * 3], [[0.0] * 3], np.zeros(13))

    rng = np.random.default_rng(11)
    O = rng.uniform(0.05, 0.95, (4000, 3))
    O[:, 2] = rng.uniform(0.05, 2.0, 4000)
    D = rng.normal(size=(4000, 3))
    meshes = [(desc.meshes[k].vertices, desc.meshes[k].faces) for k in names]
    frames = [d.frame for d in desc.instances]
    for ray_mask in (FULL_MASK, 0x3, 0xF0):
        got = closest_hit_batch(tl, O, D, ray_mask=ray_mask)
        ref = oracle_for(meshes, frames).closest_hit_batch(O, D, ray_mask=ray_mask)
        # origins inside the box, t down to ~1e-3: fp32 t carries ~ulp(|o|) absolute error
        same, _ = _agree(got, ref, t_abs=8 * 2.0 ** -23)
        _only_ties(got, ref)
    # deform the cube BLAS (refit) and move the second cube instance, then refresh
    cube = names.index("cube")
    newv = desc.meshes["cube"].vertices * np.array([1.2, 0.8, 1.1])
    blases[cube].refit(vertices=newv)
    with pytest.raises(RuntimeError, match="refresh_instance_bounds"):
        closest_hit_batch(tl, O, D)
    insts[5].frame = SrtFrame(np.array([0.25, 0.4, 0.25]), np.array([0.0, 1.0, 0.0]), 0.3,
                              np.array([0.55, 0.05, 0.6]))
    tl.refresh_instance_bounds()
    meshes[cube] = (newv, desc.meshes["cube"].faces)
    frames[5] = insts[5].frame
    got = closest_hit_batch(tl, O, D)
    ref = oracle_for(meshes, frames).closest_hit_batch(O, D)
    same, both = _agree(got, ref, t_abs=8 * 2.0 ** -23)
    _only_ties(got, ref)
    assert np.allclose(got[5][both], ref[5][both], atol=1e-12)
    assert np.isin(5, got[1])                               # the moved instance is hit


def test_tlas_api_errors(native):
    b = Blas.from_mesh([[0, 0, 0], [1, 0, 0], [0, 1, 0]], [[0, 1, 2]])
    with pytest.raises(ValueError):
        Tlas([], [b])
    with pytest.raises(ValueError):
        Tlas([Instance(3)], [b])
    with pytest.raises(ValueError):
        Blas.from_mesh([[0, 0, 0]], np.zeros((0, 3), np.int64))
    with pytest.raises(ValueError):
        Instance(0, mask=1 << 33)
    with pytest.raises(ValueError):
        b.refit(vertices=np.zeros((4, 3)))
    tl = Tlas([Instance(0), Instance(0, SrtFrame(translation=np.array([0.0, 0.0, 2.0])))], [b])
    t, inst, prim = closest_hit_batch(tl, [[0.2, 0.2, 5.0]], [[0.0, 0.0, -1.0]])[:3]
    assert inst[0] == 1 and prim[0] == 0 and abs(t[0] - 3.0) < 1e-6
    # exact tie between two coincident instances: the lower instance wins (accel.py:815-817)
    tl2 = Tlas([Instance(0), Instance(0)], [b])
    assert closest_hit_batch(tl2, [[0.2, 0.2, 5.0]], [[0.0, 0.0, -1.0]])[1][0] == 0


@pytest.mark.parametrize("which", ["cornell", "spheres"])
def test_compile_two_level_queries_and_render(native, which):
    """compile_scene(two_level=True): queries through the two-level kernels, frames through
    the device flatten of the same Tlas -- both against the reference's goldens."""
    from paper_2603_00292_b200 import IntegratorConfig, compile_scene, render_frame
    desc = scenes.cornell_description() if which == "cornell" else scenes.spheres_description()
    sc = compile_scene(desc, two_level=True)
    assert isinstance(sc.tlas, Tlas) and sc.render_tlas is not None
    if which == "cornell":
        g = golden("cornell_hits")
        res = closest_hit_batch(sc, g["O"], g["D"])
        same, _ = _agree(res, tuple(g[k] for k in ("t", "inst", "prim", "u", "v", "n")))
        assert same.all()
        r = golden("cornell_render")
        jobs = [("eye32", "eye"), ("pt24", "pt"), ("nee16", "pt-nee")]
        for name, integ in jobs:
            w, h, spp, seed, jit, md = (int(x) for x in r[name + "_args"])
            acc, st = render_frame(sc, w, h, spp, integ, seed=seed, cfg=IntegratorConfig(max_depth=md),
                                   jitter=bool(jit), return_stats=True)
            d = acc.mean() - r[name][:, :, :3] / r[name][:, :, 3:]
            assert float(np.sqrt(np.mean(d ** 2))) <= 1e-4, name
            assert st["rays"] == int(r[name + "_rays"]), name
    else:
        g = golden("spheres")
        res = closest_hit_batch(sc, g["O"], g["D"], registry=sc.registry)
        same, _ = _agree(res, tuple(g["p_" + k] for k in ("t", "inst", "prim", "u", "v", "n")))
        assert same.all()
        for name, integ in (("eye", "eye"), ("pt", "pt"), ("nee", "pt-nee")):
            w, h, spp, md = (int(x) for x in g["render_" + name + "_args"])
            acc, st = render_frame(sc, w, h, spp, integ, cfg=IntegratorConfig(max_depth=md), return_stats=True)
            d = acc.mean() - g["render_" + name][:, :, :3] / g["render_" + name][:, :, 3:]
            assert float(np.sqrt(np.mean(d ** 2))) <= 1e-4, name
            assert st["rays"] == int(g["render_" + name + "_rays"]), name


def test_flatten_refill_after_refit(native):
    """Tlas.flatten(into=...) re-makes the render copy after a Blas refit + refresh."""
    from paper_2603_00292_b200 import IntegratorConfig, compile_scene, render_frame
    desc = scenes.cornell_description()
    tl, blases, insts, _ = tlas_from_description(desc)
    mats = list(desc.materials)
    inst_mat = np.array([mats.index(d.material) for d in desc.instances], np.int32)
    mc = np.array([desc.materials[k].color for k in mats])
    me = np.array([desc.materials[k].emissive for k in mats])
    flat = tl.flatten(inst_mat, mc, me)
    cube = list(desc.meshes).index("cube")
    blases[cube].refit(vertices=desc.meshes["cube"].vertices * 1.5)
    with pytest.raises(RuntimeError):
        tl.flatten(inst_mat, mc, me, into=flat)
    tl.refresh_instance_bounds()
    tl.flatten(inst_mat, mc, me, into=flat)
    # the refilled flat scene traces like the two-level one
    rng = np.random.default_rng(5)
    O = rng.uniform(0.05, 0.95, (3000, 3))
    D = rng.normal(size=(3000, 3))
    a = closest_hit_batch(flat, O, D)
    b = closest_hit_batch(tl, O, D)
    _only_ties(a, b)
