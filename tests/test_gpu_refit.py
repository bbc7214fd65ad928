"""Device refits of a flat scene against fresh compiles of the same geometry.

* Scene.refit_mesh (Blas.refit(vertices), accel.py:263-283): the device kernel's world
  triangles and world normals are bit-identical to compile_scene's host computation, for
  every instance of the mesh (SRT frames included), and so is the rebuilt LBVH; the light
  table follows an emissive mesh;
* GpuTlas.refit (world triangle rows): the world normals follow the new triangles.
"""

import dataclasses

import numpy as np
import pytest

from paper_2603_00292_b200 import closest_hit_batch, compile_scene, render_frame, scenes

pytestmark = pytest.mark.gpu


def _with_vertices(desc, name, V):
    meshes = dict(desc.meshes)
    meshes[name] = dataclasses.replace(meshes[name], vertices=V)
    return dataclasses.replace(desc, meshes=meshes)


def _rays(n, seed, lo, hi):
    rng = np.random.default_rng(seed)
    O = rng.uniform(lo, hi, (n, 3))
    D = rng.normal(size=(n, 3))
    return O, D


def _same_scene(a, b, O, D):
    assert np.array_equal(a.tlas.tris, b.tlas.tris)
    da, db = a.tlas.download(), b.tlas.download()
    for k in da:
        assert np.array_equal(da[k], db[k]), k
    ha, hb = closest_hit_batch(a, O, D), closest_hit_batch(b, O, D)
    for x, y in zip(ha, hb):
        assert np.array_equal(x, y, equal_nan=True)


def test_refit_mesh_instanced_srt(native):
    """Cornell's cube mesh is instanced twice with rotated, scaled frames."""
    desc = scenes.cornell_description()
    sc = compile_scene(desc)
    rng = np.random.default_rng(2)
    V = desc.meshes["cube"].vertices * 1.3 + rng.normal(scale=0.02, size=desc.meshes["cube"].vertices.shape)
    sc.refit_mesh("cube", V)
    O, D = _rays(20000, 1, 0.05, 0.95)
    _same_scene(sc, compile_scene(_with_vertices(desc, "cube", V)), O, D)
    # back to the original vertices: the compile-time scene again
    sc.refit_mesh("cube", desc.meshes["cube"].vertices)
    _same_scene(sc, compile_scene(desc), O, D)


@pytest.mark.parametrize("f32", [False, True])
def test_refit_mesh_config2_sphere(native, f32):
    desc = scenes.sphere_description(100, 200)
    sc = compile_scene(desc)
    V = desc.meshes["mesh"].vertices * np.array([1.0, 0.7, 1.2])
    if f32:      # fp32 input is widened exactly: the same scene as its float64 values
        V = V.astype(np.float32)
    sc.refit_mesh("mesh", V, bits=63)
    ref = compile_scene(_with_vertices(desc, "mesh", V.astype(np.float64)), "lbvh63")
    _same_scene(sc, ref, *_rays(20000, 3, -2, 2))
    a = render_frame(sc, 64, 48, 1, "eye", seed=1)
    b = render_frame(ref, 64, 48, 1, "eye", seed=1)
    assert np.array_equal(a.data, b.data)


def test_refit_mesh_emissive_updates_lights(native):
    desc = scenes.cornell_description()
    sc = compile_scene(desc)
    V = desc.meshes["lightquad"].vertices + np.array([0.05, -0.02, 0.03])
    sc.refit_mesh("lightquad", V)
    ref = compile_scene(_with_vertices(desc, "lightquad", V))
    for f in ("v0", "v1", "v2", "normal", "emissive", "area"):
        assert np.array_equal(getattr(sc.lights, f), getattr(ref.lights, f)), f
    a = render_frame(sc, 32, 32, 2, "pt-nee", seed=5)
    b = render_frame(ref, 32, 32, 2, "pt-nee", seed=5)
    assert np.array_equal(a.data, b.data)


def test_refit_mesh_errors(native):
    desc = scenes.cornell_description()
    sc = compile_scene(desc)
    with pytest.raises(ValueError, match="vertex count changed"):
        sc.refit_mesh("cube", np.zeros((3, 3)))
    with pytest.raises(ValueError, match="unknown mesh"):
        sc.refit_mesh("nope", np.zeros((3, 3)))
    two = compile_scene(desc, two_level=True)
    with pytest.raises(ValueError, match="flat scene"):
        two.refit_mesh("cube", desc.meshes["cube"].vertices)


def test_tlas_refit_world_rows_updates_normals(native):
    """Identity instance with fp32-representable vertices: world rows == local vertices, so
    the device normals of GpuTlas.refit equal compile_scene's of the new mesh."""
    desc = scenes.sphere_description(40, 80)
    V0 = desc.meshes["mesh"].vertices.astype(np.float32).astype(np.float64)
    desc = _with_vertices(desc, "mesh", V0)
    sc = compile_scene(desc)
    V = (V0 * np.array([1.5, 0.8, 1.1])).astype(np.float32).astype(np.float64)
    F = desc.meshes["mesh"].faces
    sc.tlas.refit(V[F].reshape(-1, 9).astype(np.float32))
    _same_scene(sc, compile_scene(_with_vertices(desc, "mesh", V)), *_rays(5000, 4, -2, 2))


def test_two_level_blas_refit_equals_fresh_blas(native):
    """Blas.refit runs the device kernel (local rows + float64 local normals); the refitted
    two-level scene answers every query exactly like one built from the new vertices."""
    from paper_2603_00292_b200 import Blas, Instance, build_tlas
    desc = scenes.cornell_description()
    names = list(desc.meshes)
    cube = names.index("cube")
    rng = np.random.default_rng(6)
    V = desc.meshes["cube"].vertices * np.array([1.2, 0.8, 1.1]) + rng.normal(scale=0.01, size=(8, 3))

    def tlas(cube_vertices):
        bl = [Blas.from_mesh(cube_vertices if k == "cube" else desc.meshes[k].vertices, desc.meshes[k].faces)
              for k in names]
        return bl, build_tlas([Instance(names.index(d.mesh), d.frame) for d in desc.instances], bl)

    bl, tl = tlas(desc.meshes["cube"].vertices)
    bl[cube].refit(vertices=V)
    tl.refresh_instance_bounds()
    _, ref = tlas(V)
    O, D = _rays(20000, 7, 0.05, 0.95)
    for x, y in zip(closest_hit_batch(tl, O, D), closest_hit_batch(ref, O, D)):
        assert np.array_equal(x, y, equal_nan=True)
