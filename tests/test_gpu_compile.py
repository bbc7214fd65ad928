"""compile_scene on the device (rt_mesh_upload + rt_scene_compile) against the host restatement.

The flat scene the kernels write -- fp32 world rows, float64 world normals, float64 local
rows, (inst, prim, mask, material) per flat id -- must equal oracle.flat_world (compile_scene's
numpy assembly, scene.py:79-141 with accel.py:311-336 / 843-847) bit for bit, and the
Blas.from_mesh checks (accel.py:223-236) must raise the reference's BuildError messages.
"""

import dataclasses
import time

import numpy as np
import pytest

from paper_2603_00292_b200 import BuildError, compile_scene, scenes
from paper_2603_00292_b200.frames import SrtFrame
from paper_2603_00292_b200.scene_io import InstanceDecl, TriangleMesh

pytestmark = pytest.mark.gpu


def _check_flat(oracle_mod, desc):
    sc = compile_scene(desc)
    ref = oracle_mod.flat_world(desc)
    nt = ref["tris"].shape[0]
    tris, n32, n64, local = sc.tlas.geometry()
    assert np.array_equal(tris[:nt].view(np.uint32), ref["tris"].view(np.uint32))
    assert np.array_equal(n64[:nt].view(np.uint64), ref["normals64"].view(np.uint64))   # signed zeros too
    assert np.array_equal(n32[:nt].view(np.uint32), ref["normals64"].astype(np.float32).view(np.uint32))
    assert np.array_equal(local[:nt], ref["local_rows"])
    for k in ("tri_inst", "tri_prim", "tri_mask", "tri_material"):
        assert np.array_equal(getattr(sc.tlas, k)[:nt], ref[k]), k
    return sc, ref


def test_cornell_flat_world(native, oracle_mod):
    sc, _ = _check_flat(oracle_mod, scenes.cornell_description())
    orc = oracle_mod.scene_from_description(scenes.cornell_description())
    lo, hi = orc.root_box()
    assert np.array_equal(sc.root_box[0], lo) and np.array_equal(sc.root_box[1], hi)
    assert sc.diagonal() == orc.diagonal()


def test_spheres_scene_flat_world(native, oracle_mod):
    desc = scenes.spheres_description()
    sc, ref = _check_flat(oracle_mod, desc)
    ns = len(desc.spheres)
    assert sc.tlas.n == ref["tris"].shape[0] + ns
    inst = sc.tlas.tri_inst[-ns:]
    assert np.array_equal(inst, len(desc.instances) + np.arange(ns))


def _instanced_desc(seed, n_meshes=3, n_inst=7):
    g = np.random.default_rng(seed)
    meshes = {}
    for k in range(n_meshes):
        nv = int(g.integers(5, 60))
        meshes[f"m{k}"] = TriangleMesh(g.normal(size=(nv, 3)), g.integers(0, nv, size=(int(g.integers(3, 90)), 3)))
    base = scenes.cornell_description()
    insts = []
    for i in range(n_inst):
        ax = g.normal(size=3)
        fr = SrtFrame(scale=tuple(g.uniform(0.3, 2.0, 3)), rotation_axis=tuple(ax / np.linalg.norm(ax)),
                      rotation_angle=float(g.uniform(-3, 3)), translation=tuple(g.normal(size=3)))
        insts.append(InstanceDecl(mesh=f"m{i % n_meshes}", material=list(base.materials)[i % len(base.materials)],
                                  frame=fr, mask=int(g.integers(1, 2 ** 32))))
    return dataclasses.replace(base, meshes=meshes, instances=insts, spheres=[])


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_random_srt_instances_flat_world(native, oracle_mod, seed):
    _check_flat(oracle_mod, _instanced_desc(seed))


def _one_mesh(V, F):
    return scenes.single_mesh_description(TriangleMesh(np.asarray(V, float), np.asarray(F)), (0, 0, 3), (1, 0, 0),
                                          (0, 1, 0))


def test_build_errors_match_reference_messages(native):
    V = np.random.default_rng(0).normal(size=(30, 3))
    F = np.arange(30).reshape(-1, 3)
    with pytest.raises(BuildError, match="^cannot build over zero primitives$"):
        compile_scene(_one_mesh(V, np.zeros((0, 3), np.int64)))
    for bad in (-1, 30):
        F2 = F.copy()
        F2[4, 1] = bad
        with pytest.raises(BuildError, match="^face index out of range$"):
            compile_scene(_one_mesh(V, F2))
    V2 = V.copy()
    V2[22, 2] = np.nan          # triangle 7
    V2[10, 0] = np.inf          # triangle 3: the first non-finite one is reported
    with pytest.raises(BuildError, match="^non-finite bounds for primitive 3$"):
        compile_scene(_one_mesh(V2, F))
    # an out-of-range index wins over a non-finite triangle (the reference checks it first)
    F3 = F.copy()
    F3[9, 0] = 99
    with pytest.raises(BuildError, match="^face index out of range$"):
        compile_scene(_one_mesh(V2, F3))


def test_build_error_order_and_recovery(native):
    """The meshes are validated behind the instance tables and the flat-scene kernels
    (rt_mesh_upload_async): a bad mesh still wins over a bad instance (the reference builds
    every Blas first), a failed mesh writes nothing, and the next compile is exact."""
    import dataclasses
    V = np.random.default_rng(1).normal(size=(30, 3))
    F = np.arange(30).reshape(-1, 3)
    F2 = F.copy()
    F2[6, 2] = 10 ** 9
    bad = _one_mesh(V, F2)
    bad_inst = dataclasses.replace(bad, instances=[dataclasses.replace(bad.instances[0], material="no-such")])
    with pytest.raises(BuildError, match="^face index out of range$"):
        compile_scene(bad_inst)
    with pytest.raises(KeyError):                 # a good mesh: the instance's own error
        compile_scene(dataclasses.replace(_one_mesh(V, F), instances=bad_inst.instances))
    two = dataclasses.replace(bad, meshes={"a": TriangleMesh(V, F), "mesh": bad.meshes["mesh"]})
    with pytest.raises(BuildError, match="^face index out of range$"):
        compile_scene(two)
    good = _one_mesh(V, F)
    a = compile_scene(good).tlas.geometry()
    with pytest.raises(BuildError):
        compile_scene(bad)
    b = compile_scene(good).tlas.geometry()
    for x, y in zip(a, b):
        assert np.array_equal(x, y)


def test_compile_time_config_sizes(native):
    """compile_scene from the reference's float64 / int64 host arrays:
    printed for the record (1M sphere, 10M soup)."""
    import torch
    for desc, label in ((scenes.sphere_description(), "1M sphere"), (scenes.soup_description(), "10M soup")):
        compile_scene(desc)            # warm-up (allocator, context)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        sc = compile_scene(desc)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        print(f"compile_scene({label}, lbvh30): {1e3 * dt:.1f} ms (incl. H2D of float64 vertices + int64 faces, "
              f"device validation, flatten, LBVH build)")
        assert sc.tlas.n in (1_000_000, 10_000_000)


def test_async_upload_abi(native):
    """rt_mesh_upload_async / rt_mesh_upload_finish at the C ABI: the verdict arrives at
    finish (BuildError code), a failed mesh is refused by rt_scene_compile (RT_ESTATE), a
    second finish is a no-op, and a pending mesh can be destroyed safely."""
    import ctypes
    from paper_2603_00292_b200 import _native
    L = _native.lib()
    ctx = _native.Context.get(0)
    V = np.random.default_rng(2).normal(size=(30, 3))
    F = np.arange(30, dtype=np.int64).reshape(-1, 3)
    bounds = np.zeros(6)
    m = ctypes.c_void_p()
    assert L.rt_mesh_upload_async(ctx.handle, 30, _native.ptr(V), 10, _native.ptr(F), ctypes.byref(m)) == 0
    assert L.rt_mesh_upload_finish(ctx.handle, m, _native.ptr(bounds)) == 0
    assert np.array_equal(bounds, np.concatenate([V.min(0), V.max(0)]))
    assert L.rt_mesh_upload_finish(ctx.handle, m, _native.ptr(bounds)) == 0       # again: no-op
    L.rt_mesh_destroy(m)
    F2 = F.copy()
    F2[3, 0] = 30
    bad = ctypes.c_void_p()
    assert L.rt_mesh_upload_async(ctx.handle, 30, _native.ptr(V), 10, _native.ptr(F2), ctypes.byref(bad)) == 0
    rc = L.rt_mesh_upload_finish(ctx.handle, bad, _native.ptr(bounds))
    assert rc != 0 and L.rt_last_error().decode() == "face index out of range"
    src = (_native.InstanceSrc * 1)()
    src[0].mesh, src[0].material, src[0].mask = 0, 0, 0xFFFFFFFF
    src[0].matrix[:] = [1, 0, 0, 0, 0, 1, 0, 0, 0, 0, 1, 0]
    src[0].inverse[:] = [1, 0, 0, 0, 0, 1, 0, 0, 0, 0, 1, 0]
    col = np.ones((1, 3), np.float32)
    h = ctypes.c_void_p()
    rc = L.rt_scene_compile(ctx.handle, 1, (ctypes.c_void_p * 1)(bad.value), 1, src, 0, None, _native.ptr(col),
                            _native.ptr(col), 1, ctypes.byref(h))
    assert rc != 0 and "failed its validation" in L.rt_last_error().decode()
    L.rt_mesh_destroy(bad)
    pend = ctypes.c_void_p()
    assert L.rt_mesh_upload_async(ctx.handle, 30, _native.ptr(V), 10, _native.ptr(F), ctypes.byref(pend)) == 0
    L.rt_mesh_destroy(pend)                                                    # still pending: waits
