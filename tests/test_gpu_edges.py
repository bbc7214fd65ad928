"""Edge cases the reference defines (accel.py, geometry.py) on the GPU paths, against the
float64 oracle: exact ties between coincident triangles (lowest instance, then prim),
zero-area triangles, zero / NaN directions, empty t ranges, one-triangle scenes."""

import math

import numpy as np
import pytest

from paper_2603_00292_b200 import (Blas, Instance, SrtFrame, any_hit_batch, build_tlas, closest_hit_batch,
                                   compile_scene, render_frame)
from paper_2603_00292_b200.camera import Camera
from paper_2603_00292_b200.scene_io import InstanceDecl, Material, SceneDescription, TriangleMesh

pytestmark = pytest.mark.gpu


def _desc(meshes, insts):
    cam = Camera(np.array([0.0, 0.0, 5.0]), np.array([1.0, 0.0, 0.0]), np.array([0.0, 1.0, 0.0]))
    return SceneDescription(cam, meshes, {k: k + ".obj" for k in meshes}, {"m": Material([0.5, 0.5, 0.5])}, insts, [],
                            np.zeros(3), np.zeros(3))


def _oracle(oracle_mod, desc):
    return oracle_mod.scene_from_description(desc)


@pytest.fixture(scope="module")
def tie_scene():
    # quad split into 2 triangles, duplicated inside the mesh (prims 2, 3 == 0, 1) and
    # instanced twice at the same place, plus a zero-area triangle and a far triangle
    V = np.array([[-1, -1, 0], [1, -1, 0], [1, 1, 0], [-1, 1, 0], [0, 0, 0], [0, 0, -3], [2, 0, -3], [0, 2, -3]],
                 float)
    F = np.array([[0, 1, 2], [0, 2, 3], [0, 1, 2], [0, 2, 3], [4, 4, 4], [5, 6, 7]])
    desc = _desc({"q": TriangleMesh(V, F)}, [InstanceDecl("q", "m"), InstanceDecl("q", "m")])
    return desc


def test_exact_ties_lowest_instance_then_prim(native, oracle_mod, tie_scene):
    rng = np.random.default_rng(3)
    O = np.concatenate([rng.uniform(-0.9, 0.9, (500, 2)), np.full((500, 1), 2.0)], axis=1)
    D = np.tile([[0.0, 0.0, -1.0]], (500, 1)) + rng.normal(scale=0.05, size=(500, 3))
    orc = _oracle(oracle_mod, tie_scene)
    rt, ri, rp = orc.closest_hit_batch(O, D)[:3]
    quad = (ri >= 0) & (rp != 5)                          # (prim 5: the far triangle behind the quad)
    assert quad.mean() > 0.9
    assert np.all(ri[quad] == 0) and np.all(rp[quad] <= 1)  # instance 0 and the first copy win
    for two in (False, True):
        sc = compile_scene(tie_scene, two_level=two)
        t, inst, prim = closest_hit_batch(sc, O, D)[:3]
        assert np.array_equal(inst, ri) and np.array_equal(prim, rp)
        assert np.allclose(t, rt, rtol=1e-6)


def test_degenerate_directions_and_ranges(native, oracle_mod, tie_scene):
    O = np.array([[0.2, 0.3, 2.0]] * 6)
    D = np.array([[0, 0, 0], [np.nan, 0, -1], [0, 0, -1], [0, 0, -1], [0, 0, -1], [0, 0, -1]], float)
    tmin = np.array([0, 0, 3.0, 0, 0, 0])                  # ray 2: empty range (tmin > tmax below)
    tmax = np.array([1e30, 1e30, 1.0, 1.0, 2.0, 1e30])     # ray 3: stops short; ray 4: ends exactly at the hit
    orc = _oracle(oracle_mod, tie_scene)
    rt, ri = orc.closest_hit_batch(O, D, tmin, tmax)[:2]
    sc = compile_scene(tie_scene)
    t, inst = closest_hit_batch(sc, O, D, tmin, tmax)[:2]
    assert np.array_equal(inst, ri), (inst, ri)
    assert inst[0] == -1 and inst[1] == -1 and inst[2] == -1 and inst[3] == -1 and inst[5] == 0
    assert np.array_equal(any_hit_batch(sc, O, D, tmin, tmax), orc.any_hit_batch(O, D, tmin, tmax))


def test_one_triangle_scene(native, oracle_mod):
    V = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0]], float)
    desc = _desc({"t": TriangleMesh(V, np.array([[0, 1, 2]]))},
                 [InstanceDecl("t", "m", SrtFrame(translation=np.array([-0.3, -0.3, 0.0])))])
    sc = compile_scene(desc)
    assert sc.tlas.info()["height"] >= 1
    O = np.array([[0.0, 0.0, 1.0], [0.6, 0.6, 1.0]])
    D = np.array([[0.0, 0.0, -1.0], [0.0, 0.0, -1.0]])
    t, inst, prim, u, v, n = closest_hit_batch(sc, O, D)
    rt, ri, rp, ru, rv, rn = _oracle(oracle_mod, desc).closest_hit_batch(O, D)
    assert np.array_equal(inst, ri) and np.array_equal(prim, rp) and inst[0] == 0 and inst[1] == -1
    assert abs(t[0] - rt[0]) < 1e-6 and np.allclose(n[0], rn[0])
    acc = render_frame(sc, 8, 8, 2, "eye")
    assert np.all(acc.data[:, :, 3] == 2)


def test_instanced_rotations_two_level_vs_flat(native, oracle_mod):
    """Many SRT instances (non-uniform scale, arbitrary axes) of one mesh: the two-level
    kernels (local-space rays) and the flat path agree with the float64 oracle."""
    rng = np.random.default_rng(8)
    th = np.linspace(0, 2 * math.pi, 24, endpoint=False)
    V = np.concatenate([[[0, 0, 0.5]], np.stack([np.cos(th), np.sin(th), np.zeros_like(th)], 1) * 0.5])
    F = np.array([[0, 1 + k, 1 + (k + 1) % 24] for k in range(24)])
    insts = []
    for _ in range(40):
        ax = rng.normal(size=3)
        ax /= np.linalg.norm(ax)
        insts.append(InstanceDecl("cone", "m", SrtFrame(rng.uniform(0.3, 1.5, 3), ax, float(rng.uniform(0, 6)),
                                                        rng.uniform(-3, 3, 3)), mask=int(rng.integers(1, 4))))
    desc = _desc({"cone": TriangleMesh(V, F)}, insts)
    O = rng.uniform(-4, 4, (4000, 3))
    D = rng.normal(size=(4000, 3))
    orc = _oracle(oracle_mod, desc)
    for mask in (0xFFFFFFFF, 0x1, 0x2):
        rt, ri, rp = orc.closest_hit_batch(O, D, ray_mask=mask)[:3]
        for two in (False, True):
            sc = compile_scene(desc, two_level=two)
            t, inst, prim = closest_hit_batch(sc, O, D, ray_mask=mask)[:3]
            same = (inst == ri) & (prim == rp)
            assert same.mean() >= 0.9999, (two, mask, same.mean())
            ok = same & (ri >= 0)
            assert np.mean(np.abs(t[ok] - rt[ok]) > 1e-5 * np.abs(rt[ok]) + 8 * 2.0 ** -23) <= 1e-3
