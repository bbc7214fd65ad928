"""K1-K5: the GPU LBVH is bit-identical to the CPU restatement (oracle Part B).

Morton keys (via the sorted key sequence), the stable sort order, the Karras
topology (children, parents), the refit boxes and node heights must all match
exactly, for 30- and 63-bit keys, including heavy duplicate-key inputs (the
config-2 UV sphere has ~32% duplicate 30-bit keys).
"""

import numpy as np
import pytest

from paper_2603_00292_b200 import compile_scene, scenes

pytestmark = pytest.mark.gpu


def _gpu_vs_cpu(oracle_mod, desc, bits):
    sc = compile_scene(desc, f"lbvh{bits}")
    got = sc.tlas.download()
    lb = oracle_mod.lbvh_build(sc.tlas.tris, bits)
    for k in ("centroid_bounds", "inv_ext", "sorted_keys", "order", "child", "parent", "boxes", "height"):
        assert np.array_equal(got[k], lb[k]), k
    info = sc.tlas.info()
    assert info["height"] == lb["depth"]
    assert np.array_equal(info["root_box"], lb["root_box"])
    return sc, lb


@pytest.mark.parametrize("bits", [30, 63])
def test_cornell(native, oracle_mod, bits):
    _gpu_vs_cpu(oracle_mod, scenes.cornell_description(), bits)


@pytest.mark.parametrize("bits", [30, 63])
@pytest.mark.parametrize("size", [(3, 4), (50, 100), (500, 1000)])
def test_uv_sphere(native, oracle_mod, bits, size):
    sc, lb = _gpu_vs_cpu(oracle_mod, scenes.sphere_description(*size), bits)
    keys = lb["sorted_keys"]
    assert np.all(keys[1:] >= keys[:-1])


@pytest.mark.parametrize("bits", [30, 63])
@pytest.mark.parametrize("n", [1, 2, 3, 4097, 100_000])
def test_soup(native, oracle_mod, bits, n):
    desc = scenes.soup_description(n, seed=n)
    if n == 1:
        sc = compile_scene(desc, f"lbvh{bits}")
        assert sc.tlas.info()["height"] == 1
        return
    _gpu_vs_cpu(oracle_mod, desc, bits)


def test_all_duplicate_keys(native, oracle_mod):
    """Every centroid identical: the topology comes entirely from the index fallback."""
    from paper_2603_00292_b200.scene_io import TriangleMesh
    n = 5000
    V = np.tile(np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0]], float), (n, 1))
    mesh = TriangleMesh(V, np.arange(3 * n).reshape(-1, 3))
    desc = scenes.single_mesh_description(mesh, (0.3, 0.3, 2), (0.5, 0, 0), (0, 0.5, 0))
    sc, lb = _gpu_vs_cpu(oracle_mod, desc, 30)
    assert np.all(lb["sorted_keys"] == lb["sorted_keys"][0])
    assert np.array_equal(lb["order"], np.arange(n))
    assert lb["depth"] <= 14


def test_rebuild_is_deterministic(native):
    sc = compile_scene(scenes.soup_description(50_000, seed=1))
    a = sc.tlas.download()
    for _ in range(3):
        sc.tlas.build(30, timed=True)
        b = sc.tlas.download()
        for k in a:
            assert np.array_equal(a[k], b[k]), k
    assert sc.tlas.build_ms > 0


def test_rebuild_alternating_widths_1m(native):
    """Config-2 size, rebuilt in place with alternating Morton widths: every rebuild equals a
    fresh build (the global climb's slot records from the previous build, or a sibling's
    record that has not landed yet, must never be consumed; this caught a spin loop that
    ptxas had reduced to a single reload)."""
    desc = scenes.sphere_description()
    fresh = {b: compile_scene(desc, f"lbvh{b}").tlas.download() for b in (30, 63)}
    sc = compile_scene(desc, "lbvh30")
    for bits in (63, 30, 63, 63, 30, 30, 63, 30):
        sc.tlas.build(bits)
        got = sc.tlas.download()
        for k in fresh[bits]:
            assert np.array_equal(got[k], fresh[bits][k]), (bits, k)


def test_lbvh_cost_through_reference_traversal(native, oracle_mod):
    """the GPU BVH, traversed by the (restated) reference kernels,
    gives the SAH tree's exact hits; also reports its per-ray node/tri cost."""
    desc = scenes.sphere_description(100, 200)
    sc = compile_scene(desc, "lbvh30")
    got = sc.tlas.download()
    got["root_box"] = sc.tlas.info()["root_box"]
    got["depth"] = int(got["height"][0])
    nodes = oracle_mod.lbvh_as_reference_nodes(got, sc.tlas.n)
    mesh = desc.meshes["mesh"]
    orc_lbvh = oracle_mod.OracleScene([(mesh.vertices, mesh.faces)], [(0, 0, np.ones(3), np.array([0, 1., 0]), 0.0,
                                                                         np.zeros(3), 0xFFFFFFFF)],
                                      [[0.8] * 3], [[0.0] * 3], oracle_mod.camera13((0, 0, 2.5), (0.8, 0, 0),
                                                                                     (0, 0.45, 0)),
                                      blas_nodes=[nodes])
    orc_sah = oracle_mod.scene_from_description(desc)
    g = np.random.default_rng(0)
    O = np.tile([0.0, 0.0, 2.5], (20000, 1))
    D = np.c_[g.uniform(-0.6, 0.6, (20000, 2)), -np.ones(20000)]
    a = orc_lbvh.closest_hit_batch(O, D, with_stats=True)
    b = orc_sah.closest_hit_batch(O, D, with_stats=True)
    for x, y in zip(a[:6], b[:6]):
        assert np.array_equal(x, y)
