"""SPEC acceptance criteria checked directly on the GPU paths.

* AC1: 10^5 random ray/triangle pairs against a float64
  Moller-Trumbore: the same verdicts on the traversed fp32 rays, and t within 1e-5 (1 + |t|)
  of MT on the float64 rays (the host API refines the hit in float64).  The pairs are laid out as one scene of
  10^5 triangles, each in its own unit cell 10 apart, with ray i starting in cell i and
  limited to t <= 5, so every ray can only meet its own triangle.
* AC8: the path-traced estimate converges like 1/spp: the MSE against
  a high-spp frame drops ~4x per 4x samples, and repeated runs are bit-identical.
"""

import numpy as np
import pytest

from paper_2603_00292_b200 import IntegratorConfig, closest_hit_batch, compile_scene, render_frame, scenes
from paper_2603_00292_b200.scene_io import TriangleMesh

pytestmark = pytest.mark.gpu


def _moller_trumbore(o, d, a, b, c):
    """float64, two-sided; t (or nan on a miss), per row."""
    e1, e2 = b - a, c - a
    p = np.cross(d, e2)
    det = np.einsum("ij,ij->i", e1, p)
    with np.errstate(divide="ignore", invalid="ignore"):
        inv = 1.0 / det
        s = o - a
        u = np.einsum("ij,ij->i", s, p) * inv
        q = np.cross(s, e1)
        v = np.einsum("ij,ij->i", d, q) * inv
        t = np.einsum("ij,ij->i", e2, q) * inv
    hit = (np.abs(det) > 1e-12) & (u >= 0) & (v >= 0) & (u + v <= 1) & (t >= 0)
    return np.where(hit, t, np.nan), u, v


def test_ac1_random_pairs_vs_moller_trumbore(native):
    rng = np.random.default_rng(11)
    n = 100_000
    cells = np.stack([np.arange(n) % 100, (np.arange(n) // 100) % 100, np.arange(n) // 10_000], 1) * 10.0
    V = (cells[:, None, :] + rng.uniform(0.0, 1.0, (n, 3, 3))).reshape(-1, 3)
    V = V.astype(np.float32).astype(np.float64)                  # the GPU holds fp32 vertices
    F = np.arange(3 * n).reshape(n, 3)
    desc = scenes.single_mesh_description(TriangleMesh(V, F), (0, 0, -5), (1, 0, 0), (0, 1, 0))
    sc = compile_scene(desc)
    tri = V.reshape(n, 3, 3)
    # aim most rays at a point inside their triangle (hits), the rest anywhere (mostly misses)
    w = rng.dirichlet(np.ones(3), n)
    target = np.einsum("ij,ijk->ik", w, tri)
    O = cells + rng.uniform(-0.5, 1.5, (n, 3)) * np.array([1, 1, 1])
    O = np.where((rng.random(n) < 0.85)[:, None], O, cells + 0.5)
    D = np.where((rng.random(n) < 0.9)[:, None], target - O, rng.normal(size=(n, 3)))
    D /= np.linalg.norm(D, axis=1, keepdims=True)
    # t_max 5 keeps every ray inside its cell: its own triangle is within ~3, any other >= 7
    t, inst, prim = closest_hit_batch(sc, O, D, t_max=5.0)[:3]
    hit = prim >= 0
    assert np.all(prim[hit] == np.arange(n)[hit])                # only its own triangle
    # (a) verdicts: MT on the ray the GPU actually traverses (the API rounds rays to fp32)
    #     gives the same hit / miss on every pair
    O32, D32 = O.astype(np.float32).astype(np.float64), D.astype(np.float32).astype(np.float64)
    tr32, _, _ = _moller_trumbore(O32, D32, tri[:, 0], tri[:, 1], tri[:, 2])
    hit32 = ~np.isnan(np.where(tr32 <= 5.0, tr32, np.nan))
    assert hit32.mean() > 0.5
    assert (hit == hit32).mean() >= 0.99999, (hit == hit32).mean()
    # (b) values: the host API recomputes (t, u, v) of the hit triangle in float64 with the
    #     reference's formula on the caller's float64 ray, so t meets AC1's bound against MT
    #     on those rays; only pairs the float64 test rejects (grazing / edge) keep fp32 values
    tr, ur, vr = _moller_trumbore(O, D, tri[:, 0], tri[:, 1], tri[:, 2])
    hit64 = ~np.isnan(np.where(tr <= 5.0, tr, np.nan))
    both = hit & hit64
    within = np.abs(t[both] - tr[both]) <= 1e-5 * (1 + np.abs(tr[both]))
    assert within.mean() >= 0.9999, within.mean()
    exact = np.abs(t[both] - tr[both]) <= 1e-12 * (1 + np.abs(tr[both]))
    assert exact.mean() >= 0.999, exact.mean()
    # (c) verdicts against the float64 rays differ only where the fp32 rounding of the ray
    #     itself flips a grazing / edge-adjacent pair (34 of 10^5 here)
    assert (hit == hit64).mean() >= 0.999, (hit == hit64).mean()


def test_ac8_mse_falls_like_one_over_spp(native):
    sc = compile_scene(scenes.cornell_description())
    cfg = IntegratorConfig(max_depth=5)
    W = H = 48
    truth = render_frame(sc, W, H, 2048, "pt", seed=100, cfg=cfg).mean()
    mse = []
    for spp in (4, 16, 64):
        a = render_frame(sc, W, H, spp, "pt", seed=7, cfg=cfg)
        b = render_frame(sc, W, H, spp, "pt", seed=7, cfg=cfg)
        assert np.array_equal(a.data, b.data)                    # AC9: bit-identical reruns
        mse.append(float(np.mean((a.mean() - truth) ** 2)))
    r1, r2 = mse[0] / mse[1], mse[1] / mse[2]
    assert 2.5 < r1 < 6.0 and 2.5 < r2 < 6.0, (mse, r1, r2)
