"""Custom primitives on the GPU: spheres.scn (sphere instances behind the registry,
accel.py:366-423, scene.py:101-112) against the reference's own outputs
(tests/golden/spheres.npz) and the float64 oracle.

The sphere test runs in float64 on the device from the fp32 ray, so sphere
hits agree with the reference to ~1e-7 relative; triangle hits keep the
fp32 watertight bar.  Same bars as test_gpu_trace / test_gpu_render.
"""

import numpy as np
import pytest
import torch

from paper_2603_00292_b200 import (IntegratorConfig, IntersectorRegistry, RegistryError, any_hit_batch,
                                   closest_hit_batch, compile_scene, make_sphere_registry, render_frame, scenes)
from paper_2603_00292_b200.accel import SPHERE_GEOM_TYPE, trace_closest
from rt_helpers import golden

pytestmark = pytest.mark.gpu

T_REL = 1e-5
ID_AGREE = 0.9999


@pytest.fixture(scope="module")
def spheres_gpu(native):
    return compile_scene(scenes.spheres_description())


@pytest.fixture(scope="module")
def spheres_oracle(oracle_mod):
    return oracle_mod.scene_from_description(scenes.spheres_description())


def _check(res, g, pre, n_rays, t_abs=0.0, t_outliers=1e-4):
    t, inst, prim, u, v, n = res[:6]
    same = (inst == g[pre + "inst"]) & (prim == g[pre + "prim"])
    agree = same.mean()
    assert agree >= ID_AGREE, f"ID agreement {agree:.6f} of {n_rays}: {np.nonzero(~same)[0][:8]}"
    both = same & (inst >= 0)
    rt = g[pre + "t"]
    rel = np.maximum(np.abs(t[both] - rt[both]) - t_abs, 0) / np.abs(rt[both])
    assert np.mean(rel > T_REL) <= t_outliers, rel.max()
    sph = both & (inst >= 2)                         # sphere instances 2, 3, 4
    assert sph.sum() > 100
    assert np.all(u[sph] == 0.0) and np.all(v[sph] == 0.0)     # accel.py:621-623
    assert np.allclose(n[both], g[pre + "n"][both], atol=1e-5)
    assert np.all(t[inst < 0] == -1.0)
    return agree


def test_spheres_primary_hits(spheres_gpu):
    g = golden("spheres")
    res = closest_hit_batch(spheres_gpu, g["O"], g["D"], registry=spheres_gpu.registry)
    assert _check(res, g, "p_", g["O"].shape[0]) == 1.0


def test_spheres_random_rays_closest_and_any(spheres_gpu):
    g = golden("spheres")
    res = closest_hit_batch(spheres_gpu, g["RO"], g["RD"], g["tmin"], g["tmax"], registry=spheres_gpu.registry)
    # origins sit inside the ~[-3, 3] box: fp32 t carries ~ulp(|o|) absolute error, and
    # the fp32-rounded origin of a grazing sphere hit moves t by ~ulp(|o|) / cos
    _check(res, g, "r_", g["RO"].shape[0], t_abs=8 * 2.0 ** -23, t_outliers=1e-3)
    anyh = any_hit_batch(spheres_gpu, g["RO"], g["RD"], g["tmin"], g["tmax"], registry=spheres_gpu.registry)
    assert np.mean(anyh == g["r_any"]) >= ID_AGREE


def test_registry_contract(spheres_gpu):
    g = golden("spheres")
    # registry=None: a ray that reaches a sphere raises the reference's error (accel.py:1011-1014)
    with pytest.raises(RegistryError, match="geometry type 0 and ray type 0") as ei:
        closest_hit_batch(spheres_gpu, g["O"], g["D"])
    assert str(ei.value) == str(g["noreg_error"]).split(": ", 1)[1]
    with pytest.raises(RegistryError):
        any_hit_batch(spheres_gpu, g["O"], g["D"], registry=IntersectorRegistry())
    # rays that never reach a sphere succeed without a registry (the error is raised on reach)
    up = np.tile([[0.0, 5.0, 0.0]], (16, 1))
    t = closest_hit_batch(spheres_gpu, up, np.tile([[0.0, 1.0, 0.0]], (16, 1)))[0]
    assert np.all(t == -1.0)
    # a registry for another ray type does not cover ray type 0
    reg1 = make_sphere_registry(spheres_gpu.tlas.sphere_rows[:, 12:16], ray_types=(1,))
    with pytest.raises(RegistryError, match="ray type 0"):
        closest_hit_batch(spheres_gpu, g["O"], g["D"], registry=reg1)
    ok = closest_hit_batch(spheres_gpu, g["O"], g["D"], ray_type=1, registry=reg1)
    assert np.array_equal(ok[1], g["p_inst"])
    # a non-builtin intersection function has no GPU kernel and no CPU fallback
    bad = IntersectorRegistry()
    bad.register(SPHERE_GEOM_TYPE, 0, lambda *a: (-1.0, 0.0, 0.0, 0.0), spheres_gpu.tlas.sphere_rows[:, 12:16])
    with pytest.raises(RegistryError, match="no CPU fallback"):
        closest_hit_batch(spheres_gpu, g["O"], g["D"], registry=bad)
    # the device error flag was cleared: the next call succeeds
    assert closest_hit_batch(spheres_gpu, g["O"], g["D"], registry=spheres_gpu.registry)[1].max() >= 2


def test_device_trace_matches_host_api(spheres_gpu):
    g = golden("spheres")
    rays = torch.zeros((g["O"].shape[0], 8), dtype=torch.float32, device="cuda")
    rays[:, 0:3] = torch.from_numpy(g["O"]).float()
    rays[:, 4:7] = torch.from_numpy(g["D"]).float()
    rays[:, 7] = 1e30
    hits = torch.empty((rays.shape[0], 4), dtype=torch.float32, device="cuda")
    trace_closest(spheres_gpu, rays, hits)
    ids = hits[:, 1].view(torch.int32).cpu().numpy()
    host = closest_hit_batch(spheres_gpu, g["O"], g["D"], registry=spheres_gpu.registry)
    flat_inst = np.where(ids >= 0, spheres_gpu.tlas.tri_inst[np.maximum(ids, 0)], -1)
    assert np.array_equal(flat_inst, host[1])


def test_spheres_eye_vs_reference(spheres_gpu):
    g = golden("spheres")
    w, h, spp, md = (int(x) for x in g["render_eye_args"])
    acc, st = render_frame(spheres_gpu, w, h, spp, "eye", return_stats=True)
    assert st["rays"] == int(g["render_eye_rays"])
    same = np.all(np.abs(acc.data - g["render_eye"]) <= 1e-6 * np.maximum(1, np.abs(g["render_eye"])), axis=2)
    assert same.mean() == 1.0


@pytest.mark.parametrize("name", ["pt", "ao", "nee"])
def test_spheres_integrators_vs_reference(spheres_gpu, name):
    g = golden("spheres")
    w, h, spp, md = (int(x) for x in g["render_" + name + "_args"])
    integ = {"pt": "pt", "ao": "ao", "nee": "pt-nee"}[name]
    acc, st = render_frame(spheres_gpu, w, h, spp, integ, cfg=IntegratorConfig(max_depth=md, ao_ray_count=8),
                           return_stats=True)
    ref = g["render_" + name]
    d = acc.mean() - ref[:, :, :3] / ref[:, :, 3:]
    rmse = float(np.sqrt(np.mean(d ** 2)))
    assert rmse <= 1e-4, rmse
    assert np.abs(d).max() <= 1e-2
    assert st["rays"] == int(g["render_" + name + "_rays"])


def test_spheres_mega_equals_wavefront_and_oracle(spheres_gpu, spheres_oracle):
    cfg = IntegratorConfig(max_depth=5)
    a = render_frame(spheres_gpu, 96, 72, 4, "pt", cfg=cfg, kernel="mega")
    b = render_frame(spheres_gpu, 96, 72, 4, "pt", cfg=cfg, kernel="wavefront")
    assert np.array_equal(a.data, b.data)
    ref, _ = spheres_oracle.render_frame(96, 72, 4, "pt", max_depth=5, workers=8)
    d = a.mean() - ref[:, :, :3] / ref[:, :, 3:]
    assert float(np.sqrt(np.mean(d ** 2))) <= 1e-4
