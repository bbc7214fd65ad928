"""Scene state after edits, concurrent callers, and the t-window edges of the host query.

* refit_mesh moves the scene's root box (and so the default normal offset) like the
  reference's Blas.refit + refresh_instance_bounds (accel.py:263-283, 477-497; Scene.diagonal
  reads tlas.root_box live, scene.py:45-48): the refitted scene renders exactly like a fresh
  compile of the new geometry;
* a two-level scene's render copy follows Tlas.refresh_instance_bounds (the reference
  re-flattens its bundle there, accel.py:497);
* closest_hit_batch from several host threads on one device equals the serial results
  (ctypes releases the GIL; the library serialises calls per context);
* hits at the edges of [t_min, t_max) follow the reference (fp32 window rounding).
"""

import dataclasses
import threading

import numpy as np
import pytest

from paper_2603_00292_b200 import closest_hit_batch, compile_scene, render_frame, scenes
from paper_2603_00292_b200.frames import SrtFrame

pytestmark = pytest.mark.gpu


def _with_vertices(desc, name, V):
    meshes = dict(desc.meshes)
    meshes[name] = dataclasses.replace(meshes[name], vertices=V)
    return dataclasses.replace(desc, meshes=meshes)


def test_refit_mesh_moves_root_box_and_normal_offset(native):
    desc = scenes.cornell_description()
    sc = compile_scene(desc)
    # grow the walls: the scene's bounds (so its diagonal and normal offset) change
    V = desc.meshes["walls"].vertices * 1.7 - 0.2
    sc.refit_mesh("walls", V)
    fresh = compile_scene(_with_vertices(desc, "walls", V))
    assert np.array_equal(sc.root_box[0], fresh.root_box[0]) and np.array_equal(sc.root_box[1], fresh.root_box[1])
    assert sc.diagonal() == fresh.diagonal()
    a = render_frame(sc, 48, 32, 2, "pt", seed=3)
    b = render_frame(fresh, 48, 32, 2, "pt", seed=3)
    assert np.array_equal(a.data, b.data)
    # fp32 refit input (the config-2 bench path) gives the same bounds as float64
    sc.refit_mesh("walls", V.astype(np.float32))
    fresh32 = compile_scene(_with_vertices(desc, "walls", V.astype(np.float32).astype(np.float64)))
    assert sc.diagonal() == fresh32.diagonal()


def test_two_level_render_follows_refresh(native):
    desc = scenes.cornell_description()
    two = compile_scene(desc, two_level=True)
    # eye colours the white cubes like the white walls behind them: path tracing sees them
    before = render_frame(two, 40, 40, 2, "pt", seed=1)
    names = list(desc.meshes)
    cube = names.index("cube")
    newv = desc.meshes["cube"].vertices * np.array([1.4, 0.6, 1.2])
    two.tlas.blases[cube].refit(vertices=newv)
    two.tlas.instances[5].frame = SrtFrame(np.array([0.25, 0.4, 0.25]), np.array([0.0, 1.0, 0.0]), 0.3,
                                           np.array([0.55, 0.05, 0.6]))
    two.tlas.refresh_instance_bounds()
    after = render_frame(two, 40, 40, 2, "pt", seed=1)
    # the same edit as a fresh flat compile
    insts = list(desc.instances)
    insts[5] = dataclasses.replace(insts[5], frame=two.tlas.instances[5].frame)
    fresh = compile_scene(dataclasses.replace(_with_vertices(desc, "cube", newv), instances=insts))
    ref = render_frame(fresh, 40, 40, 2, "pt", seed=1)
    assert not np.array_equal(before.data, after.data)
    assert np.array_equal(after.data, ref.data)
    assert two.diagonal() == fresh.diagonal()


def test_concurrent_queries_one_device(native):
    scs = [compile_scene(scenes.sphere_description(100, 200)), compile_scene(scenes.soup_description(50_000, seed=3))]
    rng = np.random.default_rng(5)
    jobs = []
    for k in range(8):
        O = rng.uniform(-0.2, 0.2, (40_000, 3)) + np.array([0.0, 0.0, 2.5])
        D = np.c_[rng.uniform(-0.6, 0.6, (40_000, 2)), -np.ones(40_000)]
        jobs.append((scs[k % 2], O, D))
    serial = [closest_hit_batch(sc, O, D) for sc, O, D in jobs]
    out = [None] * len(jobs)

    def run(i):
        for _ in range(3):
            sc, O, D = jobs[i]
            out[i] = closest_hit_batch(sc, O, D)

    th = [threading.Thread(target=run, args=(i,)) for i in range(len(jobs))]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for a, b in zip(serial, out):
        for x, y in zip(a, b):
            assert np.array_equal(x, y)


def test_t_window_edges_match_reference(native, cornell_oracle):
    """The back wall (z = 0) seen from z = 2.4 along -z: t = 2.4 exactly in float64 (fp32(2.4)
    is 2.4000000954).  The reference's closest-hit window is [t_min, t_max): a hit at exactly
    t_max loses the scene-level test (t == best_t needs inst < best_inst = -1, accel.py:771-773,
    815-817).  Windows within an ulp of the hit must give the reference's answers, although
    they round to the same fp32 value as the hit."""
    sc = compile_scene(scenes.cornell_description())
    O = np.array([[0.5, 0.9, 2.4]])
    D = np.array([[0.0, 0.0, -1.0]])
    below, above = np.nextafter(2.4, 0.0), np.nextafter(2.4, 3.0)
    cases = [{}, {"t_max": below}, {"t_max": 2.4}, {"t_max": above}, {"t_min": below}, {"t_min": 2.4},
             {"t_min": above}]
    for kw in cases:
        g = closest_hit_batch(sc, O, D, **kw)
        r = cornell_oracle.closest_hit_batch(O, D, **kw)
        assert g[1][0] == r[1][0] and g[2][0] == r[2][0] and g[0][0] == r[0][0], (kw, g[:3], r[:3])
    assert closest_hit_batch(sc, O, D)[0][0] == 2.4
    assert closest_hit_batch(sc, O, D, t_max=2.4)[1][0] == -1
