"""compile_scene on the GPU: flatten instances, upload, build the LBVH.

Mirrors scene.py:79-141 of the reference (``compile_scene(desc, quality)`` ->
``Scene``) with ``quality`` selecting the GPU LBVH ("lbvh30" default,
"lbvh63"; the reference's "balanced"/"fast" SAH qualities map to lbvh30).
Instances are flattened on the host into world-space fp32 triangles in
(instance, prim) order, so the reference tie rule (lowest instance, then
lowest prim; accel.py:629, 815-817) is "lowest flat id" on the device.  The
per-triangle world normal is computed reference-style in float64 (local
cross product and normalisation as in geometry.py:235-237, 274-275, then the
inverse-transpose sum and renormalisation of accel.py:843-847) and only then
rounded to fp32, which preserves the signed zeros the ONB depends on.
"""

import ctypes
import math
from dataclasses import dataclass

import numpy as np

from . import _native
from ._native import BuildError, check, lib, ptr
from .accel import IntersectorRegistry, SPHERE_GEOM_TYPE, sphere_data, sphere_intersector
from .camera import Camera
from .frames import frame_to_matrix, invert_affine

QUALITIES = {"lbvh30": 30, "lbvh63": 63, "balanced": 30, "fast": 30}


@dataclass
class LightTable:
    """World-space emissive triangles (sampling.py:217-253); kept for NEE ("next")."""

    v0: np.ndarray
    v1: np.ndarray
    v2: np.ndarray
    normal: np.ndarray
    emissive: np.ndarray
    area: np.ndarray
    instance: np.ndarray
    prim: np.ndarray

    def __len__(self):
        return self.v0.shape[0]


class GpuTlas:
    """Device-resident flattened scene + LBVH (replaces Tlas/TlasBundle, accel.py:439-549)."""

    def __init__(self, ctx, tris, normals, tri_inst, tri_prim, tri_mask, tri_material, mat_color,
                 mat_emissive, bits=30, root_lo=None, root_hi=None, instances=None, inverses=None, spheres=None):
        self.ctx = ctx
        self.n = int(tris.shape[0])
        self.bits = bits
        self._tris = np.ascontiguousarray(tris, np.float32).reshape(-1, 9)
        normals64 = np.ascontiguousarray(normals, np.float64).reshape(-1, 3)
        self.normals = np.ascontiguousarray(normals64, np.float32)
        self.tri_inst = np.ascontiguousarray(tri_inst, np.int32)
        self.tri_prim = np.ascontiguousarray(tri_prim, np.int32)
        self.tri_mask = np.ascontiguousarray(tri_mask, np.uint32)
        self.tri_material = np.ascontiguousarray(tri_material, np.int32)
        self.inverses = inverses
        self.n_instances = instances
        self.world_root = (root_lo, root_hi)
        mc = np.ascontiguousarray(mat_color, np.float32).reshape(-1, 3)
        me = np.ascontiguousarray(mat_emissive, np.float32).reshape(-1, 3)
        h = ctypes.c_void_p()
        check(lib().rt_scene_create(ctx.handle, self.n, ptr(self._tris), ptr(self.normals), ptr(self.tri_inst),
                                    ptr(self.tri_prim), ptr(self.tri_mask), ptr(self.tri_material), ptr(mc),
                                    ptr(me), mc.shape[0], ctypes.byref(h)))
        self.handle = h
        # the float64 world normals themselves, for the host query's outputs
        check(lib().rt_scene_set_normals64(ctx.handle, h, ptr(normals64)))
        self.build_ms = None
        # custom primitives: the last rows of `tris` are sphere instance boxes
        self.sphere_rows = np.zeros((0, 16)) if spheres is None else np.ascontiguousarray(spheres, np.float64)
        self.n_spheres = int(self.sphere_rows.shape[0])
        if self.n_spheres:
            check(lib().rt_scene_set_spheres(ctx.handle, h, self.n_spheres, ptr(self.sphere_rows)))
        self.build(bits)

    def custom_geom_types(self):
        """accel.py Tlas.custom_geom_types: geometry types of the custom BLASes present."""
        return [SPHERE_GEOM_TYPE] if self.n_spheres else []

    def build(self, bits=None, timed=False):
        """(Re)build the LBVH from the resident triangles; returns device ms if timed."""
        bits = self.bits if bits is None else bits
        ms = ctypes.c_float(-1.0)
        check(lib().rt_bvh_build(self.ctx.handle, self.handle, bits, ctypes.byref(ms) if timed else None))
        self.bits = bits
        if timed:
            self.build_ms = ms.value
            return ms.value
        return None

    @property
    def tris(self):
        """(n, 9) fp32 world triangle rows (read back from the device after a device refit)."""
        if self._tris is None:
            t = np.empty((self.n, 9), np.float32)
            check(lib().rt_scene_get_vertices(self.ctx.handle, self.handle, ptr(t)))
            self._tris = t
        return self._tris

    def refit(self, tris, bits=None):
        """New world vertices for the same triangles (Blas.refit, accel.py:263-283): H2D, the
        world normals recomputed on the device from them, rebuild."""
        tris = np.ascontiguousarray(tris, np.float32).reshape(-1, 9)
        if tris.shape[0] != self.n:
            raise ValueError(f"triangle count changed ({self.n} -> {tris.shape[0]})")
        check(lib().rt_scene_set_vertices(self.ctx.handle, self.handle, ptr(tris)))
        check(lib().rt_scene_update_normals(self.ctx.handle, self.handle))
        self._tris = tris
        self.build(bits)

    @classmethod
    def from_handle(cls, ctx, handle, n, bits, sphere_rows=None):
        """Wrap a scene built on the device (rt_tlas_flatten); host geometry copies absent."""
        self = cls.__new__(cls)
        self.ctx, self.handle, self.n, self.bits = ctx, handle, int(n), bits
        self._tris = self.normals = self.tri_inst = self.tri_prim = self.tri_mask = self.tri_material = None
        self.inverses = self.n_instances = None
        self.world_root = (None, None)
        self.build_ms = None
        self.sphere_rows = np.zeros((0, 16)) if sphere_rows is None else sphere_rows
        self.n_spheres = int(self.sphere_rows.shape[0])
        return self

    def build_profiled(self, bits=None):
        """Rebuild with stage events; returns dict of device ms per stage."""
        bits = self.bits if bits is None else bits
        ms = np.zeros(6, np.float32)
        check(lib().rt_bvh_build_profiled(self.ctx.handle, self.handle, bits, ptr(ms)))
        self.bits = bits
        return dict(zip(("bounds", "morton_hist", "unused", "radix_passes", "slot_init", "emit_refit"), map(float, ms)))

    def info(self):
        root = np.empty(6, np.float32)
        h = ctypes.c_int32()
        ni = ctypes.c_int64()
        check(lib().rt_bvh_info(self.ctx.handle, self.handle, ptr(root), ctypes.byref(h), ctypes.byref(ni)))
        return {"root_box": root, "height": h.value, "n_internal": ni.value}

    def download(self):
        """Full LBVH for parity checks (same layout as oracle.lbvh_build)."""
        n = self.n
        m = max(n - 1, 0)
        out = {"sorted_keys": np.empty(n, np.uint64), "order": np.empty(n, np.uint32),
               "child": np.empty((m, 2), np.int32), "parent": np.empty(max(2 * n - 1, 1), np.int32),
               "boxes": np.empty((m, 12), np.float32), "height": np.empty(m, np.int32),
               "centroid_bounds": np.empty(6, np.float32), "inv_ext": np.empty(3, np.float32)}
        check(lib().rt_bvh_download(self.ctx.handle, self.handle, ptr(out["sorted_keys"]), ptr(out["order"]),
                                    ptr(out["child"]), ptr(out["parent"]), ptr(out["boxes"]), ptr(out["height"]),
                                    ptr(out["centroid_bounds"]), ptr(out["inv_ext"]), None))
        return out

    def __del__(self):
        try:
            if getattr(self, "handle", None) and _native._lib is not None:
                _native._lib.rt_scene_destroy(self.handle)
        except Exception:
            pass


@dataclass
class Scene:
    """scene.py:30-48; ``tlas`` is device-backed."""

    camera: Camera
    tlas: GpuTlas
    registry: IntersectorRegistry
    mat_color: np.ndarray
    mat_emissive: np.ndarray
    inst_material: np.ndarray
    lights: LightTable
    sky: np.ndarray
    background: np.ndarray
    root_box: tuple
    render_tlas: object = None   # two-level scenes: the device-flattened structure rt_render walks
    _meshes: dict = None         # flat scenes: mesh name -> _MeshRefit (device refit_mesh)
    _light_src: tuple = None     # (desc, material index, instances) the light table came from

    def diagonal(self) -> float:
        d = self.root_box[1] - self.root_box[0]
        return math.sqrt(float(d @ d))

    def refit_mesh(self, name, vertices, bits=None):
        """Blas.refit(vertices) (accel.py:263-283) for every instance of mesh `name` of a flat
        scene, on the device: the vertices go up (float64, or float32 as given: 24 or 12 B per
        vertex; the faces stay resident), one kernel writes the instances' world triangles and world normals exactly
        as compile_scene does on the host, and the LBVH is rebuilt.  The scene's root
        box and normal offset keep their compile-time values, as the reference's Scene does."""
        if self.render_tlas is not None or self._meshes is None:
            raise ValueError("refit_mesh needs a flat scene (two-level scenes refit their Blas)")
        if name not in self._meshes:
            raise ValueError(f"unknown mesh {name!r}")
        mr = self._meshes[name]
        # float32 input goes up as is (half the bytes) and is widened exactly on the device
        f32 = isinstance(vertices, np.ndarray) and vertices.dtype == np.float32
        V = np.ascontiguousarray(vertices, np.float32 if f32 else np.float64).reshape(-1, 3)
        if V.shape[0] != mr.nv:
            raise ValueError(f"vertex count changed ({mr.nv} -> {V.shape[0]})")
        tl = self.tlas
        check(lib().rt_scene_refit_mesh(tl.ctx.handle, tl.handle, mr.handle(tl.ctx), mr.nv, ptr(V), 1 if f32 else 0))
        tl._tris = None                          # the host copy is read back on demand
        desc, mat_index, inst_list = self._light_src
        if any(desc.materials[d.material].has_emission for d, _ in inst_list if d.mesh == name):
            # emissive instances of this mesh: the light table follows the new vertices
            import dataclasses
            meshes = dict(desc.meshes)
            meshes[name] = dataclasses.replace(meshes[name], vertices=V.astype(np.float64))
            self._light_src = (dataclasses.replace(desc, meshes=meshes), mat_index, inst_list)
            self.lights = _light_rows(self._light_src[0], mat_index, inst_list)
            rows = np.ascontiguousarray(np.concatenate([self.lights.v0, self.lights.v1, self.lights.v2,
                                                        self.lights.normal, self.lights.emissive,
                                                        self.lights.area[:, None]], axis=1), np.float32)
            check(lib().rt_scene_set_lights(tl.ctx.handle, tl.handle, rows.shape[0], ptr(rows)))
        tl.build(bits)


class _MeshRefit:
    """One mesh of a flat scene for Scene.refit_mesh: faces + instance frames, uploaded on
    first use (rt_mesh_create)."""

    def __init__(self, nv, faces, inst, flags=0):
        self.nv = int(nv)
        self.flags = int(flags)
        self.faces = np.ascontiguousarray(faces, np.int32).reshape(-1, 3)
        # rows of 21 doubles: the 3x4 matrix, then the 3x3 block of its inverse
        self.xform = np.ascontiguousarray([np.concatenate([m.reshape(12), inv[:, :3].reshape(9)]) for m, inv, _ in inst],
                                          np.float64)
        self.offset = np.ascontiguousarray([o for _, _, o in inst], np.int64)
        self._h = None

    def handle(self, ctx):
        if self._h is None:
            h = ctypes.c_void_p()
            check(lib().rt_mesh_create(ctx.handle, self.nv, self.faces.shape[0], ptr(self.faces), len(self.offset),
                                       ptr(self.xform), ptr(self.offset), self.flags, ctypes.byref(h)))
            self._h = h
        return self._h

    def __del__(self):
        try:
            if self._h and _native._lib is not None:
                _native._lib.rt_mesh_destroy(self._h)
        except Exception:
            pass


def _local_normals(V, F):
    """geometry.py:229-237, 274-275 per face, float64, reference operation order."""
    a, b, c = V[F[:, 0]], V[F[:, 1]], V[F[:, 2]]
    e0 = b - a
    e1 = c - b
    nx = e0[:, 1] * e1[:, 2] - e0[:, 2] * e1[:, 1]
    ny = e0[:, 2] * e1[:, 0] - e0[:, 0] * e1[:, 2]
    nz = e0[:, 0] * e1[:, 1] - e0[:, 1] * e1[:, 0]
    with np.errstate(invalid="ignore", divide="ignore"):
        nlen = np.sqrt(nx * nx + ny * ny + nz * nz)
        return nx / nlen, ny / nlen, nz / nlen


def _world_normals(inv, lnx, lny, lnz):
    """accel.py:843-847: inverse-transpose sum, then multiply by 1/sqrt."""
    wnx = inv[0, 0] * lnx + inv[1, 0] * lny + inv[2, 0] * lnz
    wny = inv[0, 1] * lnx + inv[1, 1] * lny + inv[2, 1] * lnz
    wnz = inv[0, 2] * lnx + inv[1, 2] * lny + inv[2, 2] * lnz
    with np.errstate(invalid="ignore", divide="ignore"):
        inv_len = 1.0 / np.sqrt(wnx * wnx + wny * wny + wnz * wnz)
    return np.stack([wnx * inv_len, wny * inv_len, wnz * inv_len], axis=1)


def _light_rows(desc, mats_index, inst_list):
    """scene.py:58-76."""
    rows = []
    for i, (decl, m) in enumerate(inst_list):
        mat = desc.materials[decl.material]
        if not mat.has_emission:
            continue
        mesh = desc.meshes[decl.mesh]
        world = mesh.vertices @ m[:, :3].T + m[:, 3]
        for prim, (i0, i1, i2) in enumerate(mesh.faces):
            w0, w1, w2 = world[i0], world[i1], world[i2]
            n = np.cross(w1 - w0, w2 - w1)
            nlen = math.sqrt(float(n @ n))
            if nlen == 0.0:
                continue
            rows.append((w0, w1, w2, n / nlen, mat.emissive, 0.5 * nlen, i, prim))
    if not rows:
        z = np.zeros((0, 3))
        return LightTable(z, z, z, z, z, np.zeros(0), np.zeros(0, np.int64), np.zeros(0, np.int64))
    col = lambda k: np.array([r[k] for r in rows])
    return LightTable(col(0).reshape(-1, 3), col(1).reshape(-1, 3), col(2).reshape(-1, 3), col(3).reshape(-1, 3),
                      col(4).reshape(-1, 3), col(5), col(6).astype(np.int64), col(7).astype(np.int64))


def compile_scene(desc, quality: str = "lbvh30", device: int = 0, two_level: bool = False) -> Scene:
    """Flatten + upload + LBVH build (scene.py:79-141 semantics, GPU backend).

    two_level=True builds the reference's structure instead -- one device Blas per mesh
    (and per sphere), a Tlas over the instances -- so queries run the two-level kernels;
    rendering walks a flattened copy made on the device from that Tlas."""
    if quality not in QUALITIES:
        raise ValueError(f"unknown build quality {quality!r}, expected one of {tuple(QUALITIES)}")
    if two_level:
        return _compile_two_level(desc, quality, device)
    mat_names = list(desc.materials)
    mat_index = {n: i for i, n in enumerate(mat_names)}
    mat_color = np.array([desc.materials[n].color for n in mat_names]).reshape(-1, 3)
    mat_emissive = np.array([desc.materials[n].emissive for n in mat_names]).reshape(-1, 3)
    if not desc.instances and not desc.spheres:
        raise BuildError("a scene needs at least one instance")

    # per-mesh validation and local data (Blas.from_mesh, accel.py:223-236)
    mesh_cache = {}
    for name, mesh in desc.meshes.items():
        V = np.ascontiguousarray(mesh.vertices, np.float64).reshape(-1, 3)
        F = np.ascontiguousarray(mesh.faces, np.int64).reshape(-1, 3)
        if F.shape[0] == 0:
            raise BuildError("cannot build over zero primitives")
        if F.min() < 0 or F.max() >= V.shape[0]:
            raise BuildError("face index out of range")
        tri = V[F]
        lo, hi = tri.min(axis=1), tri.max(axis=1)
        bad = ~np.isfinite(lo).all(axis=1) | ~np.isfinite(hi).all(axis=1)
        if bad.any():
            raise BuildError(f"non-finite bounds for primitive {int(np.argmax(bad))}")
        mesh_cache[name] = (V, F, lo.min(axis=0), hi.max(axis=0), _local_normals(V, F))

    tris, normals, t_inst, t_prim, t_mask, t_mat = [], [], [], [], [], []
    local_rows = []                # float64 local vertices per flat primitive (the query's refinement)
    inst_material, inst_list, inverses = [], [], []
    wlo, whi = [], []
    mesh_inst = {}                 # mesh name -> [(3x4 matrix, inverse, first flat triangle)]
    off = 0
    for i, decl in enumerate(desc.instances):
        V, F, rlo, rhi, ln = mesh_cache[decl.mesh]
        m = frame_to_matrix(decl.frame)
        try:
            inv = invert_affine(m)
        except ValueError as exc:
            raise BuildError(f"instance {i} frame is not invertible") from exc
        mesh_inst.setdefault(decl.mesh, []).append((m, inv, off))
        off += F.shape[0]
        inverses.append(inv)
        inst_list.append((decl, m))
        # world AABB of the 8 root-box corners (accel.py:459-469)
        corners = np.array([[(rlo, rhi)[s & 1][0], (rlo, rhi)[(s >> 1) & 1][1], (rlo, rhi)[(s >> 2) & 1][2]]
                            for s in range(8)])
        pts = corners @ m[:, :3].T + m[:, 3]
        wlo.append(pts.min(axis=0))
        whi.append(pts.max(axis=0))
        W = (m[0, 0] * V[:, 0:1] + m[0, 1] * V[:, 1:2] + m[0, 2] * V[:, 2:3] + m[0, 3],
             m[1, 0] * V[:, 0:1] + m[1, 1] * V[:, 1:2] + m[1, 2] * V[:, 2:3] + m[1, 3],
             m[2, 0] * V[:, 0:1] + m[2, 1] * V[:, 1:2] + m[2, 2] * V[:, 2:3] + m[2, 3])
        Wv = np.concatenate(W, axis=1)
        tris.append(Wv[F].reshape(-1, 9).astype(np.float32))
        local_rows.append(V[F].reshape(-1, 9))
        normals.append(_world_normals(inv, *ln))       # float64; GpuTlas keeps both widths
        nt = F.shape[0]
        t_inst.append(np.full(nt, i, np.int32))
        t_prim.append(np.arange(nt, dtype=np.int32))
        t_mask.append(np.full(nt, decl.mask, np.uint32))
        mi = mat_index[decl.material]
        inst_material.append(mi)
        t_mat.append(np.full(nt, mi, np.int32))
    # sphere instances after the mesh instances (scene.py:101-112): one custom
    # primitive each, flat ids after every triangle; its leaf box is the world AABB
    # of the transformed local box (accel.py:459-469), rounded outward to fp32
    sph_rows = []
    if desc.spheres:
        rows = np.array([[*sph.center, sph.radius] for sph in desc.spheres], dtype=np.float64)
        sphere_data(rows)                               # radius > 0 (accel.py:403-408)
        for k, sph in enumerate(desc.spheres):
            m = frame_to_matrix(sph.frame)
            try:
                inv = invert_affine(m)
            except ValueError as exc:
                raise BuildError(f"sphere {k} frame is not invertible") from exc
            c, r = rows[k, :3], rows[k, 3]
            blo, bhi = c - r, c + r
            corners = np.array([[(blo, bhi)[s & 1][0], (blo, bhi)[(s >> 1) & 1][1], (blo, bhi)[(s >> 2) & 1][2]]
                                for s in range(8)])
            pts = corners @ m[:, :3].T + m[:, 3]
            lo, hi = pts.min(axis=0), pts.max(axis=0)
            wlo.append(lo)
            whi.append(hi)
            lo32 = lo.astype(np.float32)
            hi32 = hi.astype(np.float32)
            lo32 = np.where(lo32.astype(np.float64) > lo, np.nextafter(lo32, np.float32(-np.inf)), lo32)
            hi32 = np.where(hi32.astype(np.float64) < hi, np.nextafter(hi32, np.float32(np.inf)), hi32)
            tris.append(np.concatenate([lo32, hi32, lo32]).reshape(1, 9).astype(np.float32))
            normals.append(np.zeros((1, 3)))
            local_rows.append(np.zeros((1, 9)))
            inst_idx = len(desc.instances) + k
            t_inst.append(np.array([inst_idx], np.int32))
            t_prim.append(np.zeros(1, np.int32))
            t_mask.append(np.array([sph.mask], np.uint32))
            mi = mat_index[sph.material]
            inst_material.append(mi)
            t_mat.append(np.array([mi], np.int32))
            inverses.append(inv)
            sph_rows.append(np.concatenate([inv.reshape(12), c, [r]]))
    root_lo = np.min(np.array(wlo), axis=0)
    root_hi = np.max(np.array(whi), axis=0)
    ctx = _native.Context.get(device)
    tlas = GpuTlas(ctx, np.concatenate(tris), np.concatenate(normals), np.concatenate(t_inst),
                   np.concatenate(t_prim), np.concatenate(t_mask), np.concatenate(t_mat), mat_color, mat_emissive,
                   bits=QUALITIES[quality], root_lo=root_lo, root_hi=root_hi,
                   instances=len(desc.instances) + len(desc.spheres), inverses=np.array(inverses),
                   spheres=np.array(sph_rows) if sph_rows else None)
    inv12 = np.ascontiguousarray(np.array(inverses, np.float64).reshape(-1, 12))
    check(lib().rt_scene_set_local_frames(ctx.handle, tlas.handle, inv12.shape[0], ptr(inv12),
                                          ptr(np.ascontiguousarray(np.concatenate(local_rows), np.float64))))
    registry = IntersectorRegistry()
    if desc.spheres:
        registry.register(SPHERE_GEOM_TYPE, 0, sphere_intersector,
                          np.array([[*sph.center, sph.radius] for sph in desc.spheres]))
    lights = _light_rows(desc, mat_index, inst_list)
    if len(lights):
        rows = np.ascontiguousarray(np.concatenate([lights.v0, lights.v1, lights.v2, lights.normal, lights.emissive,
                                                    lights.area[:, None]], axis=1), np.float32)
        check(lib().rt_scene_set_lights(ctx.handle, tlas.handle, rows.shape[0], ptr(rows)))
    sc = Scene(camera=desc.camera, tlas=tlas, registry=registry, mat_color=mat_color, mat_emissive=mat_emissive,
               inst_material=np.array(inst_material, np.int64), lights=lights,
               sky=np.ascontiguousarray(desc.sky, np.float64), background=np.ascontiguousarray(desc.background,
                                                                                               np.float64),
               root_box=(root_lo, root_hi))
    sc._meshes = {name: _MeshRefit(mesh_cache[name][0].shape[0], mesh_cache[name][1], inst)
                  for name, inst in mesh_inst.items()}
    sc._light_src = (desc, mat_index, inst_list)
    return sc


def _compile_two_level(desc, quality, device):
    """compile_scene through Blas / Instance / Tlas (scene.py:85-117), plus the device flatten."""
    from .twolevel import Blas, Instance, Tlas
    from .accel import sphere_aabbs
    if not desc.instances and not desc.spheres:
        raise BuildError("a scene needs at least one instance")
    mat_names = list(desc.materials)
    mat_index = {n: i for i, n in enumerate(mat_names)}
    mat_color = np.array([desc.materials[n].color for n in mat_names]).reshape(-1, 3)
    mat_emissive = np.array([desc.materials[n].emissive for n in mat_names]).reshape(-1, 3)
    blases, blas_of_mesh, instances, inst_material, inst_list = [], {}, [], [], []
    for name, mesh in desc.meshes.items():
        blas_of_mesh[name] = len(blases)
        blases.append(Blas.from_mesh(mesh.vertices, mesh.faces, quality, device=device))
    for decl in desc.instances:
        instances.append(Instance(blas_of_mesh[decl.mesh], decl.frame, decl.mask))
        inst_material.append(mat_index[decl.material])
        inst_list.append((decl, frame_to_matrix(decl.frame)))
    registry = IntersectorRegistry()
    if desc.spheres:
        rows = np.array([[*sph.center, sph.radius] for sph in desc.spheres], dtype=np.float64)
        registry.register(SPHERE_GEOM_TYPE, 0, sphere_intersector, sphere_data(rows))
        for i, sph in enumerate(desc.spheres):
            instances.append(Instance(len(blases), sph.frame, sph.mask))
            blases.append(Blas.from_aabbs(sphere_aabbs(rows[i:i + 1]), SPHERE_GEOM_TYPE, quality, data_offset=i,
                                          device=device))
            inst_material.append(mat_index[sph.material])
    tlas = Tlas(instances, blases, quality)
    flat = tlas.flatten(np.array(inst_material, np.int32), mat_color, mat_emissive, registry, QUALITIES[quality])
    lights = _light_rows(desc, mat_index, inst_list)
    if len(lights):
        rows = np.ascontiguousarray(np.concatenate([lights.v0, lights.v1, lights.v2, lights.normal, lights.emissive,
                                                    lights.area[:, None]], axis=1), np.float32)
        check(lib().rt_scene_set_lights(flat.ctx.handle, flat.handle, rows.shape[0], ptr(rows)))
    return Scene(camera=desc.camera, tlas=tlas, registry=registry, mat_color=mat_color, mat_emissive=mat_emissive,
                 inst_material=np.array(inst_material, np.int64), lights=lights,
                 sky=np.ascontiguousarray(desc.sky, np.float64),
                 background=np.ascontiguousarray(desc.background, np.float64), root_box=tlas.root_box,
                 render_tlas=flat)
