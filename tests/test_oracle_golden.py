"""Pin the float64 oracle (oracle/rt_oracle.c) to the reference's own outputs.

Every fixture in tests/golden/ was produced by the reference package
(tests/golden/make_golden.py).  The oracle restates the reference operation
for operation, so these comparisons are exact (==), not tolerances.
"""

import numpy as np
import pytest

from rt_helpers import golden


def test_pcg_streams_and_kat(oracle_mod):
    g = golden("pcg")
    for (sd, px, s), u, (st, inc) in zip(g["streams"], g["uniforms"], g["states"]):
        ost, oinc = oracle_mod.stream_for(int(sd), int(px), int(s))
        assert (ost, oinc) == (int(st), int(inc))
        assert np.array_equal(oracle_mod.uniforms(int(sd), int(px), int(s), 8), u)
    # SURVEY 8(c) known answer
    assert oracle_mod.stream_for(0, 0, 0) == (0x8a40023040a62ab7, 0xc510c17fe888c66b)
    assert list(g["kat_u32"]) == [0xa15c02b7, 0x7b47f409, 0xba1d3330, 0x83d2f293, 0xbfa4784b, 0xcbed606e]


def test_tri_hit_matches_reference(oracle_mod):
    g = golden("tri_hit")
    out = np.array([oracle_mod.tri_hit(o, d, 0.0, 1e30, a, b, c)
                    for o, d, a, b, c in zip(g["o"], g["d"], g["v0"], g["v1"], g["v2"])])
    assert np.array_equal(out, g["out"])
    assert out[0, 0] == 1.0
    assert out[1, 0] < 0.0           # SPEC.md:70 parallel ray misses


@pytest.mark.parametrize("tag", ["soup", "sphere"])
@pytest.mark.parametrize("quality", ["balanced", "fast"])
def test_sah_build_bit_exact(oracle_mod, tag, quality):
    g = golden("bvh_sah")
    nd = oracle_mod.build_bvh(g[tag + "_lo"], g[tag + "_hi"], quality)
    for k in ("bounds", "left", "right", "count", "axis", "order"):
        assert np.array_equal(nd[k], g[f"{tag}_{quality}_{k}"]), k
    assert nd["depth"] == int(g[f"{tag}_{quality}_depth"])


def test_cornell_scene_assembly(cornell_oracle):
    g = golden("cornell_hits")
    sc = cornell_oracle
    assert np.array_equal(sc.inverses, g["meta_inverses"])
    assert np.array_equal(sc.matrices, g["meta_matrices"])
    assert np.array_equal(sc.camera, g["meta_cam"])
    assert sc.diagonal() == float(g["meta_diag"])
    for k in ("lv0", "lv1", "lv2", "ln", "lemis", "larea"):
        assert np.array_equal(getattr(sc, k), g["meta_" + k]), k


def test_cornell_closest_hits_bit_exact(cornell_oracle):
    g = golden("cornell_hits")
    t, inst, prim, u, v, n, stats = cornell_oracle.closest_hit_batch(g["O"], g["D"], with_stats=True)
    for a, b in ((t, "t"), (inst, "inst"), (prim, "prim"), (u, "u"), (v, "v"), (n, "n"), (stats, "stats")):
        assert np.array_equal(a, g[b]), b


def test_cornell_random_rays_closest_any_mask(cornell_oracle):
    g = golden("cornell_hits")
    r = cornell_oracle.closest_hit_batch(g["RO"], g["RD"], g["tmin"], g["tmax"], with_stats=True, workers=3)
    for a, b in zip(r, ("rt", "ri", "rp", "ru", "rv", "rn", "rs")):
        assert np.array_equal(a, g[b]), b
    assert np.array_equal(cornell_oracle.any_hit_batch(g["RO"], g["RD"], g["tmin"], g["tmax"]), g["rany"])
    mt = cornell_oracle.closest_hit_batch(g["RO"], g["RD"], g["tmin"], g["tmax"], ray_mask=0)[0]
    assert np.array_equal(mt, g["masked_t"]) and np.all(mt < 0)


@pytest.mark.parametrize("name", ["eye32", "eye16c", "pt24", "pt16s7", "ao16", "nee16"])
def test_cornell_render_frame_bit_exact(cornell_oracle, name):
    g = golden("cornell_render")
    w, h, spp, seed, jit, md = (int(x) for x in g[name + "_args"])
    integ = {"eye": "eye", "pt2": "pt", "pt1": "pt", "ao1": "ao", "nee": "pt-nee"}[name[:3]]
    acc, rays = cornell_oracle.render_frame(w, h, spp, integ, seed=seed, workers=3, max_depth=md,
                                            ao_ray_count=8, jitter=bool(jit))
    assert rays == int(g[name + "_rays"])
    assert np.array_equal(acc, g[name])


def test_sample_split_sums_to_full_frame(cornell_oracle):
    """Sample-index split: slices [s0, s1) use the global s in the stream hash."""
    full, r0 = cornell_oracle.render_frame(12, 10, 6, "pt", max_depth=5)
    a, r1 = cornell_oracle.render_frame(12, 10, 2, "pt", max_depth=5, s0=0)
    b, r2 = cornell_oracle.render_frame(12, 10, 4, "pt", max_depth=5, s0=2)
    assert r0 == r1 + r2
    assert np.allclose(a + b, full, rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("tag", ["sphere", "soup"])
def test_synthetic_hits_bit_exact(oracle_mod, tag):
    from paper_2603_00292_b200 import scenes
    g = golden("synthetic_hits")
    desc = scenes.uv_sphere(50, 100) if tag == "sphere" else scenes.random_soup(4000, seed=0)
    cam = ((0, 0, 2.5), (0.8, 0, 0), (0, 0.45, 0)) if tag == "sphere" else \
        ((0.5, 0.5, 2.5), (0.6222, 0, 0), (0, 0.35, 0))
    sc = oracle_mod.scene_from_description(scenes.single_mesh_description(desc, *cam))
    r = sc.closest_hit_batch(g[tag + "_O"], g[tag + "_D"], with_stats=True)
    for a, k in zip(r, ("t", "inst", "prim", "u", "v", "n", "stats")):
        assert np.array_equal(a, g[f"{tag}_{k}"]), k
    acc, _ = sc.render_frame(48, 27, 1, "eye")
    assert np.array_equal(acc, g[tag + "_eye"])


def test_lbvh_through_reference_traversal(oracle_mod, reference):
    """the CPU LBVH, wrapped as a reference Blas, gives the SAH tree's exact hits."""
    from paper_2603_00292_b200 import scenes
    pt = reference
    from pathtrace.accel import Blas, Instance, Tlas, TRIANGLES
    mesh = scenes.uv_sphere(40, 80)
    tris = mesh.vertices[mesh.faces].reshape(-1, 9).astype(np.float32)
    for bits in (30, 63):
        lb = oracle_mod.lbvh_build(tris, bits)
        nodes = oracle_mod.lbvh_as_reference_nodes(lb, tris.shape[0])
        blas = Blas(nodes, TRIANGLES, vertices=mesh.vertices, faces=mesh.faces)
        tl = Tlas([Instance(0)], [blas])
        ref_blas = Blas.from_mesh(mesh.vertices, mesh.faces)
        tl_ref = Tlas([Instance(0)], [ref_blas])
        g = np.random.default_rng(5)
        O = np.tile([0.0, 0.0, 2.5], (4000, 1))
        D = np.c_[g.uniform(-0.5, 0.5, (4000, 2)), -np.ones(4000)]
        a = pt.closest_hit_batch(tl, O, D)
        b = pt.closest_hit_batch(tl_ref, O, D)
        for x, y in zip(a, b):
            assert np.array_equal(x, y)


# ---- spheres.scn: custom-primitive sphere instances (accel.py:366-423, scene.py:101-112) ----

@pytest.fixture(scope="module")
def spheres_oracle(oracle_mod):
    from paper_2603_00292_b200 import scenes
    return oracle_mod.scene_from_description(scenes.spheres_description())


def test_spheres_scene_assembly(spheres_oracle):
    g = golden("spheres")
    assert np.array_equal(spheres_oracle.inverses, g["meta_inverses"])
    assert np.array_equal(spheres_oracle.inst_material, g["meta_inst_material"])
    assert spheres_oracle.diagonal() == float(g["meta_diag"])
    assert np.array_equal(spheres_oracle.tlas_nodes["bounds"][0], g["meta_root_box"])


def test_spheres_closest_any_bit_exact(spheres_oracle):
    g = golden("spheres")
    r = spheres_oracle.closest_hit_batch(g["O"], g["D"], with_stats=True)
    for a, k in zip(r, ("t", "inst", "prim", "u", "v", "n", "stats")):
        assert np.array_equal(a, g["p_" + k]), k
    r = spheres_oracle.closest_hit_batch(g["RO"], g["RD"], g["tmin"], g["tmax"], with_stats=True, workers=3)
    for a, k in zip(r, ("t", "inst", "prim", "u", "v", "n", "stats")):
        assert np.array_equal(a, g["r_" + k]), k
    assert np.array_equal(spheres_oracle.any_hit_batch(g["RO"], g["RD"], g["tmin"], g["tmax"]), g["r_any"])
    # the fixture exercises the sphere instances (2, 3, 4) and the ground/panel meshes
    assert set(np.unique(g["r_inst"])) >= {-1, 0, 1, 2, 3, 4}


@pytest.mark.parametrize("name", ["eye", "pt", "ao", "nee"])
def test_spheres_render_frame_bit_exact(spheres_oracle, name):
    g = golden("spheres")
    w, h, spp, md = (int(x) for x in g["render_" + name + "_args"])
    integ = {"eye": "eye", "pt": "pt", "ao": "ao", "nee": "pt-nee"}[name]
    acc, rays = spheres_oracle.render_frame(w, h, spp, integ, seed=0, workers=3, max_depth=md, ao_ray_count=8)
    assert rays == int(g["render_" + name + "_rays"])
    assert np.array_equal(acc, g["render_" + name])
