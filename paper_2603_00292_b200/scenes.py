"""Built-in scenes: the bundled Cornell box and the synthetic benchmark meshes.

The Cornell box reproduces ``pkg/scenes/cornell.scn`` and its OBJ meshes
(cornell.scn:1-19) as in-memory data, so the GPU box (which has no
/root/reference) renders the same scene; tests/test_host.py checks it against
the reference's parsed description.  The synthetic meshes follow SURVEY.md
section 8(d) exactly (configs 2 and 4): float64 generation, then rounded to
fp32 so both the GPU and the float64 oracle see identical vertices.
"""

import math

import numpy as np

from .camera import Camera
from .frames import SrtFrame
from .scene_io import InstanceDecl, Material, SceneDescription, SphereDecl, TriangleMesh


def _quads(verts, quads):
    """OBJ-style quad split (i, j, k), (i, k, l) with 1-based indices."""
    faces = []
    for q in quads:
        a, b, c, d = (i - 1 for i in q)
        faces += [[a, b, c], [a, c, d]]
    return TriangleMesh(np.array(verts, dtype=np.float64), np.array(faces, dtype=np.int64))


def _cornell_meshes():
    walls = []
    for quad in (
        [(0, 0, 0), (1, 0, 0), (1, 0, 1), (0, 0, 1)],              # floor y = 0
        [(0, 0, 0), (1, 0, 0), (1, 1, 0), (0, 1, 0)],              # back wall z = 0
        [(0, 1, 0.65), (1, 1, 0.65), (1, 1, 1), (0, 1, 1)],        # ceiling strips
        [(0, 1, 0), (1, 1, 0), (1, 1, 0.35), (0, 1, 0.35)],
        [(0, 1, 0.35), (0.35, 1, 0.35), (0.35, 1, 0.65), (0, 1, 0.65)],
        [(0.65, 1, 0.35), (1, 1, 0.35), (1, 1, 0.65), (0.65, 1, 0.65)],
    ):
        walls += quad
    n = len(walls) // 4
    meshes = {
        "walls": _quads(walls, [(4 * k + 1, 4 * k + 2, 4 * k + 3, 4 * k + 4) for k in range(n)]),
        "leftwall": _quads([(0, 0, 0), (0, 1, 0), (0, 1, 1), (0, 0, 1)], [(1, 2, 3, 4)]),
        "rightwall": _quads([(1, 0, 0), (1, 1, 0), (1, 1, 1), (1, 0, 1)], [(1, 2, 3, 4)]),
        "lightquad": _quads([(0.35, 1, 0.35), (0.65, 1, 0.35), (0.65, 1, 0.65), (0.35, 1, 0.65)],
                            [(1, 2, 3, 4)]),
    }
    cube_v = [(x, y, z) for y in (0, 1) for (x, z) in ((-0.5, -0.5), (0.5, -0.5), (0.5, 0.5), (-0.5, 0.5))]
    meshes["cube"] = _quads(cube_v, [(1, 2, 3, 4), (5, 6, 7, 8), (1, 2, 6, 5), (2, 3, 7, 6),
                                     (3, 4, 8, 7), (4, 1, 5, 8)])
    return meshes


def cornell_description() -> SceneDescription:
    """cornell.scn: 6 instances over 5 meshes, 42 world triangles, one lamp."""
    meshes = _cornell_meshes()
    mats = {
        "white": Material([0.73, 0.73, 0.73]),
        "red": Material([0.63, 0.065, 0.05]),
        "green": Material([0.14, 0.45, 0.091]),
        "lamp": Material([0, 0, 0], [17, 12, 4]),
    }
    y = np.array([0.0, 1.0, 0.0])
    inst = [
        InstanceDecl("walls", "white"),
        InstanceDecl("leftwall", "red"),
        InstanceDecl("rightwall", "green"),
        InstanceDecl("lightquad", "lamp"),
        InstanceDecl("cube", "white", SrtFrame(np.array([0.3, 0.6, 0.3]), y, math.radians(15.0),
                                                 np.array([0.33, 0.0, 0.35]))),
        InstanceDecl("cube", "white", SrtFrame(np.array([0.3, 0.3, 0.3]), y, math.radians(-18.0),
                                                 np.array([0.66, 0.0, 0.64]))),
    ]
    cam = Camera(np.array([0.5, 0.5, 2.4]), np.array([0.35, 0.0, 0.0]), np.array([0.0, 0.35, 0.0]))
    return SceneDescription(cam, meshes, {k: f"{k}.obj" for k in meshes}, mats, inst, [],
                            np.zeros(3), np.zeros(3))


def furnace_description() -> SceneDescription:
    """furnace.scn: 0.5-albedo quad (scaled 100) under a unit sky."""
    quad = _quads([(-0.5, 0, -0.5), (0.5, 0, -0.5), (0.5, 0, 0.5), (-0.5, 0, 0.5)], [(1, 4, 3, 2)])
    cam = Camera(np.array([0.0, 3.0, 0.0]), np.array([0.25, 0.0, 0.0]), np.array([0.0, 0.0, -0.25]))
    return SceneDescription(cam, {"ground": quad}, {"ground": "quad.obj"}, {"gray": Material([0.5] * 3)},
                            [InstanceDecl("ground", "gray", SrtFrame(scale=np.array([100.0, 1.0, 100.0])))],
                            [], np.ones(3), np.zeros(3))


def spheres_description() -> SceneDescription:
    """spheres.scn: three custom-primitive spheres on a ground quad under an emissive
    panel (spheres.scn:1-17; quad.obj = unit quad in y = 0, face 1 4 3 2)."""
    quad = _quads([(-0.5, 0, -0.5), (0.5, 0, -0.5), (0.5, 0, 0.5), (-0.5, 0, 0.5)], [(1, 4, 3, 2)])
    mats = {
        "floor": Material([0.6, 0.6, 0.6]),
        "orange": Material([0.85, 0.45, 0.15]),
        "blue": Material([0.2, 0.35, 0.8]),
        "gray": Material([0.75, 0.75, 0.75]),
        "lamp": Material([0, 0, 0], [10, 10, 9]),
    }
    inst = [
        InstanceDecl("ground", "floor", SrtFrame(scale=np.array([40.0, 1.0, 40.0]))),
        InstanceDecl("panel", "lamp", SrtFrame(np.array([3.0, 1.0, 3.0]), np.array([1.0, 0.0, 0.0]),
                                               math.radians(180.0), np.array([0.0, 4.0, 0.0]))),
    ]
    sph = [
        SphereDecl("orange", np.zeros(3), 0.6, SrtFrame(translation=np.array([-1.3, 0.6, 0.0]))),
        SphereDecl("blue", np.zeros(3), 0.6, SrtFrame(translation=np.array([1.3, 0.6, 0.0]))),
        SphereDecl("gray", np.zeros(3), 0.9, SrtFrame(translation=np.array([0.0, 0.9, -1.6]))),
    ]
    cam = Camera(np.array([0.0, 1.2, 4.0]), np.array([0.45, 0.0, 0.0]), np.array([0.0, 0.45, 0.0]))
    sky = np.array([0.05, 0.07, 0.1])
    return SceneDescription(cam, {"ground": quad, "panel": quad}, {"ground": "quad.obj", "panel": "quad.obj"}, mats,
                            inst, sph, sky, sky.copy())


def uv_sphere(stacks=500, slices=1000):
    """(stacks*slices*2) triangles incl. zero-area pole tris; fp32-rounded."""
    th = np.pi * np.arange(stacks + 1) / stacks
    ph = 2 * np.pi * np.arange(slices) / slices
    T, P = np.meshgrid(th, ph, indexing="ij")
    V = np.stack([np.sin(T) * np.cos(P), np.cos(T), np.sin(T) * np.sin(P)], axis=-1).reshape(-1, 3)
    V = V.astype(np.float32).astype(np.float64)
    i = np.arange(stacks)[:, None]
    j = np.arange(slices)[None, :]
    a = i * slices + j
    b = i * slices + (j + 1) % slices
    c = a + slices
    d = b + slices
    F = np.stack([np.stack([a, c, b], -1), np.stack([b, c, d], -1)], axis=2).reshape(-1, 3)
    return TriangleMesh(V, F.astype(np.int64))


def random_soup(n, seed=0):
    """centroid U[0,1)^3, vertex offsets +-0.005, fp32-rounded."""
    rng = np.random.default_rng(seed)
    c = rng.random((n, 1, 3))
    e = (rng.random((n, 3, 3)) - 0.5) * 0.01
    V = (c + e).reshape(-1, 3).astype(np.float32).astype(np.float64)
    return TriangleMesh(V, np.arange(3 * n, dtype=np.int64).reshape(-1, 3))


def single_mesh_description(mesh, origin, right, up, color=(0.8, 0.8, 0.8)) -> SceneDescription:
    cam = Camera(np.asarray(origin, float), np.asarray(right, float), np.asarray(up, float))
    return SceneDescription(cam, {"mesh": mesh}, {"mesh": "<synthetic>"}, {"m": Material(list(color))},
                            [InstanceDecl("mesh", "m")], [], np.zeros(3), np.zeros(3))


def sphere_description(stacks=500, slices=1000):
    """Config 2 scene: camera origin (0,0,2.5), right (0.8,0,0), up (0,0.45,0)."""
    return single_mesh_description(uv_sphere(stacks, slices), (0, 0, 2.5), (0.8, 0, 0), (0, 0.45, 0))


def soup_description(n=10_000_000, seed=0):
    """Config 4 scene: camera origin (0.5,0.5,2.5), right (0.6222,0,0), up (0,0.35,0)."""
    return single_mesh_description(random_soup(n, seed), (0.5, 0.5, 2.5), (0.6222, 0, 0), (0, 0.35, 0))
