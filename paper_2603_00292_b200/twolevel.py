"""Two-level acceleration structures on the GPU: ``Blas``, ``Instance``, ``Tlas``.

Drop-in for the reference's accel.py:211-283 (Blas.from_mesh / from_aabbs /
refit), 339-346 (Instance), 439-549 (Tlas, refresh_instance_bounds,
custom_geom_types) and build_tlas (accel.py:552-553).  Every BLAS is a
device-resident LBVH over its LOCAL primitives; the TLAS is an LBVH over the
instance world boxes; ``closest_hit_batch`` / ``any_hit_batch`` on a ``Tlas``
run the two-level kernels of csrc/tlas.cu (local-space rays, the reference's
tie rule, float64 normals through the instance inverse transpose).

``compile_scene`` keeps using the flattened single-level structure
(scene.py here), which renders faster; this module is for callers that build
and edit instanced scenes through the reference's object API (refit a BLAS,
move an instance, refresh the top level) without re-uploading world geometry.
"""

import ctypes
import math
from dataclasses import dataclass, field

import numpy as np

from . import _native
from ._native import BuildError, RegistryError, check, host_empty, lib, ptr, t_range
from .accel import CUSTOM, SPHERE_GEOM_TYPE, TRIANGLES, _check_mask, registry_error, sphere_intersector
from .frames import FULL_MASK, SrtFrame, frame_to_matrix, invert_affine

QUALITY_BITS = {"balanced": 30, "fast": 30, "lbvh30": 30, "lbvh63": 63}


def _bits(quality):
    if quality not in QUALITY_BITS:
        raise ValueError(f"unknown build quality {quality!r}, expected one of {tuple(QUALITY_BITS)}")
    return QUALITY_BITS[quality]


def _outward_f32(lo, hi):
    """float64 boxes -> fp32 boxes that contain them (round lo down, hi up)."""
    lo32 = lo.astype(np.float32)
    hi32 = hi.astype(np.float32)
    lo32 = np.where(lo32.astype(np.float64) > lo, np.nextafter(lo32, np.float32(-np.inf)), lo32)
    hi32 = np.where(hi32.astype(np.float64) < hi, np.nextafter(hi32, np.float32(np.inf)), hi32)
    return lo32, hi32


def _local_normals64(V, F):
    """geometry.py:229-237, 274-275: unit (v1-v0) x (v2-v1) per face, float64."""
    a, b, c = V[F[:, 0]], V[F[:, 1]], V[F[:, 2]]
    e0, e1 = b - a, c - b
    nx = e0[:, 1] * e1[:, 2] - e0[:, 2] * e1[:, 1]
    ny = e0[:, 2] * e1[:, 0] - e0[:, 0] * e1[:, 2]
    nz = e0[:, 0] * e1[:, 1] - e0[:, 1] * e1[:, 0]
    with np.errstate(invalid="ignore", divide="ignore"):
        nlen = np.sqrt(nx * nx + ny * ny + nz * nz)
        return np.ascontiguousarray(np.stack([nx / nlen, ny / nlen, nz / nlen], axis=1))


class Blas:
    """Bottom-level BVH over one triangle mesh or one AABB list, resident on a GPU."""

    def __init__(self, ctx, kind, quality, vertices=None, faces=None, aabbs=None, geom_type=-1, data_offset=0):
        self.ctx = ctx
        self.kind = kind
        self.quality = quality
        self.vertices = vertices
        self.faces = faces
        self.aabbs = aabbs
        self.geom_type = int(geom_type)
        self.data_offset = int(data_offset)
        self.handle = None
        self._mesh = None          # device faces for refit (scene._MeshRefit), made on first refit
        self.version = 0
        rows = self._rows()
        n = rows.shape[0]
        h = ctypes.c_void_p()
        zero3 = np.zeros((n, 3), np.float32)
        ids = np.arange(n, dtype=np.int32)
        mats = np.zeros(3, np.float32)
        check(lib().rt_scene_create(ctx.handle, n, ptr(rows), ptr(zero3), ptr(np.zeros(n, np.int32)), ptr(ids),
                                    ptr(np.full(n, FULL_MASK, np.uint32)), ptr(np.zeros(n, np.int32)), ptr(mats),
                                    ptr(mats), 1, ctypes.byref(h)))
        self.handle = h
        if kind == TRIANGLES:
            check(lib().rt_scene_set_local_normals(ctx.handle, h, ptr(_local_normals64(vertices, faces))))
            check(lib().rt_scene_set_local_rows(ctx.handle, h, ptr(np.ascontiguousarray(vertices[faces].reshape(-1, 9)))))
        else:
            check(lib().rt_scene_set_custom(ctx.handle, h, self.geom_type, self.data_offset))
        self._build()

    # -- construction (accel.py:223-260) --------------------------------------
    @classmethod
    def from_mesh(cls, vertices, faces, quality="balanced", device=0) -> "Blas":
        _bits(quality)
        vertices = np.ascontiguousarray(vertices, dtype=np.float64).reshape(-1, 3)
        faces = np.ascontiguousarray(faces, dtype=np.int64).reshape(-1, 3)
        if faces.shape[0] == 0:
            raise BuildError("cannot build over zero primitives")
        if faces.min() < 0 or faces.max() >= vertices.shape[0]:
            raise BuildError("face index out of range")
        cls._check_finite_tris(vertices, faces)
        return cls(_native.Context.get(device), TRIANGLES, quality, vertices=vertices, faces=faces)

    @classmethod
    def from_aabbs(cls, aabbs, geom_type, quality="balanced", data_offset=0, device=0) -> "Blas":
        _bits(quality)
        aabbs = np.ascontiguousarray(aabbs, dtype=np.float64).reshape(-1, 6)
        if aabbs.shape[0] == 0:
            raise BuildError("cannot build over zero primitives")
        bad = ~np.isfinite(aabbs).all(axis=1)
        if bad.any():
            raise BuildError(f"non-finite bounds for primitive {int(np.argmax(bad))}")
        return cls(_native.Context.get(device), CUSTOM, quality, aabbs=aabbs, geom_type=geom_type,
                   data_offset=data_offset)

    @staticmethod
    def _check_finite_tris(V, F):
        tri = V[F]
        lo, hi = tri.min(axis=1), tri.max(axis=1)
        bad = ~np.isfinite(lo).all(axis=1) | ~np.isfinite(hi).all(axis=1)
        if bad.any():
            raise BuildError(f"non-finite bounds for primitive {int(np.argmax(bad))}")

    def _rows(self):
        if self.kind == TRIANGLES:
            return np.ascontiguousarray(self.vertices[self.faces].reshape(-1, 9).astype(np.float32))
        lo, hi = _outward_f32(self.aabbs[:, :3], self.aabbs[:, 3:])
        return np.ascontiguousarray(np.concatenate([lo, hi, lo], axis=1))

    def _build(self):
        check(lib().rt_bvh_build(self.ctx.handle, self.handle, _bits(self.quality), None))
        h = ctypes.c_int32()
        check(lib().rt_bvh_info(self.ctx.handle, self.handle, None, ctypes.byref(h), None))
        self._height = h.value

    # -- properties (accel.py:262-275) ----------------------------------------
    @property
    def prim_count(self) -> int:
        return self.faces.shape[0] if self.kind == TRIANGLES else self.aabbs.shape[0]

    @property
    def depth(self) -> int:
        """Height of the binary LBVH (the traversal stack bound)."""
        return self._height

    @property
    def root_box(self):
        """float64 (lo, hi) of all primitive boxes (== the reference's root node bounds)."""
        if self.kind == TRIANGLES:
            tri = self.vertices[self.faces]
            return tri.min(axis=(0, 1)), tri.max(axis=(0, 1))
        return self.aabbs[:, :3].min(axis=0), self.aabbs[:, 3:].max(axis=0)

    # -- refit (accel.py:263-283): new geometry, same primitives ---------------
    def refit(self, vertices=None, aabbs=None):
        """Deformed geometry, same primitives: upload and rebuild this LBVH on the GPU
        (a rebuild gives the same hits as the reference's box refit; hits do not depend
        on the topology).  Call ``Tlas.refresh_instance_bounds`` afterwards."""
        if self.kind == TRIANGLES:
            if vertices is None:
                raise ValueError("triangle refit needs updated vertex positions")
            vertices = np.ascontiguousarray(vertices, dtype=np.float64).reshape(-1, 3)
            if vertices.shape[0] != self.vertices.shape[0]:
                raise ValueError(f"vertex count changed ({self.vertices.shape[0]} -> {vertices.shape[0]})")
            self._check_finite_tris(vertices, self.faces)
            self.vertices = vertices
            # faces stay on the device: the vertices go up and one kernel writes the local
            # rows and float64 local normals (as _rows / _local_normals64 would, bit for bit)
            if self._mesh is None:
                from .scene import _MeshRefit
                ident = np.hstack([np.eye(3), np.zeros((3, 1))])
                self._mesh = _MeshRefit(vertices.shape[0], self.faces, [(ident, ident, 0)], flags=1)
            check(lib().rt_scene_refit_mesh(self.ctx.handle, self.handle, self._mesh.handle(self.ctx),
                                            vertices.shape[0], ptr(vertices), 0))
            self._build()
            self.version += 1
            return
        else:
            if aabbs is None:
                raise ValueError("custom refit needs updated AABBs")
            aabbs = np.ascontiguousarray(aabbs, dtype=np.float64).reshape(-1, 6)
            if aabbs.shape[0] != self.aabbs.shape[0]:
                raise ValueError(f"primitive count changed ({self.aabbs.shape[0]} -> {aabbs.shape[0]})")
            self.aabbs = aabbs
        check(lib().rt_scene_set_vertices(self.ctx.handle, self.handle, ptr(self._rows())))
        self._build()
        self.version += 1

    def __del__(self):
        try:
            if self.handle and _native._lib is not None:
                _native._lib.rt_scene_destroy(self.handle)
        except Exception:
            pass


@dataclass
class Instance:
    """accel.py:339-346."""

    blas_id: int
    frame: SrtFrame = field(default_factory=SrtFrame)
    mask: int = FULL_MASK

    def __post_init__(self):
        if not (0 <= self.mask <= FULL_MASK):
            raise ValueError("instance mask must fit in 32 bits")


class Tlas:
    """Top-level BVH over transformed instances (accel.py:439-549), on the GPU."""

    two_level = True

    def __init__(self, instances, blases, quality="balanced"):
        if len(instances) == 0:
            raise BuildError("a scene needs at least one instance")
        _bits(quality)
        self.instances = list(instances)
        self.blases = list(blases)
        self.quality = quality
        self.handle = None
        self._bound = {}
        devs = {b.ctx.device for b in self.blases}
        if len(devs) > 1:
            raise ValueError("all blases of a tlas must live on one device")
        for i, inst in enumerate(self.instances):
            if not (0 <= inst.blas_id < len(self.blases)):
                raise BuildError(f"instance {i} references unknown blas {inst.blas_id}")
        self.ctx = self.blases[self.instances[0].blas_id].ctx
        self.generation = 0          # bumped by refresh_instance_bounds (render copies follow it)
        inv, boxes = self._frames()
        handles = (ctypes.c_void_p * len(self.instances))(*[self.blases[i.blas_id].handle.value
                                                            for i in self.instances])
        masks = np.array([i.mask for i in self.instances], np.uint32)
        h = ctypes.c_void_p()
        check(lib().rt_tlas_create(self.ctx.handle, len(self.instances), handles, ptr(inv), ptr(boxes), ptr(masks),
                                   ctypes.byref(h)))
        self.handle = h
        self._versions = [b.version for b in self.blases]

    def _frames(self):
        """Matrices, inverses and world boxes (accel.py:451-472), float64."""
        n = len(self.instances)
        self.matrices = np.empty((n, 3, 4))
        self.inverses = np.empty((n, 3, 4))
        self.world_lo = np.empty((n, 3))
        self.world_hi = np.empty((n, 3))
        for i, inst in enumerate(self.instances):
            m = frame_to_matrix(inst.frame)
            try:
                self.inverses[i] = invert_affine(m)
            except ValueError as exc:
                raise BuildError(f"instance {i} frame is not invertible") from exc
            self.matrices[i] = m
            rlo, rhi = self.blases[inst.blas_id].root_box
            corners = np.array([[(rlo, rhi)[s & 1][0], (rlo, rhi)[(s >> 1) & 1][1], (rlo, rhi)[(s >> 2) & 1][2]]
                                for s in range(8)])
            pts = corners @ m[:, :3].T + m[:, 3]
            self.world_lo[i] = pts.min(axis=0)
            self.world_hi[i] = pts.max(axis=0)
        lo32, hi32 = _outward_f32(self.world_lo, self.world_hi)
        return (np.ascontiguousarray(self.inverses.reshape(n, 12)),
                np.ascontiguousarray(np.concatenate([lo32, hi32], axis=1)))

    @property
    def root_box(self):
        return self.world_lo.min(axis=0), self.world_hi.max(axis=0)

    def diagonal(self) -> float:
        lo, hi = self.root_box
        d = hi - lo
        return math.sqrt(float(d @ d))

    def custom_geom_types(self):
        return sorted({b.geom_type for b in self.blases if b.kind == CUSTOM})

    def refresh_instance_bounds(self):
        """accel.py:477-497: refit the top level after blas refits or frame edits."""
        inv, boxes = self._frames()
        check(lib().rt_tlas_update(self.ctx.handle, self.handle, ptr(inv), ptr(boxes)))
        self._versions = [b.version for b in self.blases]
        self.generation += 1

    # -- registry binding (accel.py:1002-1008 _dispatch_for) --------------------
    def _bind(self, registry, ray_type):
        if [b.version for b in self.blases] != self._versions:
            # the reference keeps tracing a stale copy until the refresh; the device
            # BLAS is rebuilt in place, so a query in between is refused instead
            raise RuntimeError("a blas was refit since the last Tlas.refresh_instance_bounds()")
        for g in self.custom_geom_types():
            e = registry.entry(g, ray_type) if registry is not None else None
            if e is not None and e[0] is not sphere_intersector:
                raise RegistryError("only the builtin sphere_intersector runs on the GPU (no CPU fallback for "
                                    "custom intersection functions)")
            data = None if e is None else np.ascontiguousarray(e[1], np.float64).reshape(-1, 4)
            key = None if data is None else (id(e[1]), data.shape[0], data.tobytes()[:64])
            if self._bound.get(g, "unset") == key:
                continue
            check(lib().rt_tlas_set_custom_data(self.ctx.handle, self.handle, g, 0 if data is None else data.shape[0],
                                                ptr(data)))
            self._bound[g] = key

    def flatten(self, inst_material, mat_color, mat_emissive, registry=None, bits=30, into=None):
        """Single-level copy of this scene made on the device, for rendering (rt_render walks
        the flat LBVH): triangle instances transformed by a kernel, custom primitives
        (spheres of the registry's data) appended.  ``into``: a previous flatten to refill."""
        from .scene import GpuTlas
        if [b.version for b in self.blases] != self._versions:
            raise RuntimeError("a blas was refit since the last Tlas.refresh_instance_bounds()")
        n_inst = len(self.instances)
        inst_material = np.ascontiguousarray(inst_material, np.int32).reshape(n_inst)
        mc = np.ascontiguousarray(mat_color, np.float32).reshape(-1, 3)
        me = np.ascontiguousarray(mat_emissive, np.float32).reshape(-1, 3)
        boxes, rows, cinst, cprim = [], [], [], []
        for i, inst in enumerate(self.instances):
            b = self.blases[inst.blas_id]
            if b.kind != CUSTOM:
                continue
            e = registry.entry(b.geom_type, 0) if registry is not None else None
            if e is None or e[0] is not sphere_intersector:
                raise RegistryError(f"no GPU intersector registered for geometry type {b.geom_type} (ray type 0)")
            data = np.asarray(e[1], np.float64).reshape(-1, 4)
            m = self.matrices[i]
            for p in range(b.prim_count):
                lo, hi = b.aabbs[p, :3], b.aabbs[p, 3:]
                corners = np.array([[(lo, hi)[s & 1][0], (lo, hi)[(s >> 1) & 1][1], (lo, hi)[(s >> 2) & 1][2]]
                                    for s in range(8)])
                pts = corners @ m[:, :3].T + m[:, 3]
                w_lo, w_hi = _outward_f32(pts.min(axis=0), pts.max(axis=0))
                boxes.append(np.concatenate([w_lo, w_hi, w_lo]))
                rows.append(np.concatenate([self.inverses[i].reshape(12), data[b.data_offset + p]]))
                cinst.append(i)
                cprim.append(p)
        nc = len(rows)
        boxes = np.ascontiguousarray(np.array(boxes, np.float32).reshape(nc, 9)) if nc else None
        rows = np.ascontiguousarray(np.array(rows, np.float64).reshape(nc, 16)) if nc else None
        cinst = np.ascontiguousarray(np.array(cinst, np.int32)) if nc else None
        cprim = np.ascontiguousarray(np.array(cprim, np.int32)) if nc else None
        h = ctypes.c_void_p(into.handle.value if into is not None else None)
        check(lib().rt_tlas_flatten(self.ctx.handle, self.handle, ptr(np.ascontiguousarray(self.matrices.reshape(-1, 12))),
                                    ptr(inst_material), ptr(mc), ptr(me), mc.shape[0], nc, ptr(boxes), ptr(rows),
                                    ptr(cinst), ptr(cprim), bits, ctypes.byref(h)))
        if into is not None:
            return into
        n = sum(self.blases[i.blas_id].prim_count for i in self.instances)
        return GpuTlas.from_handle(self.ctx, h, n, bits, rows)

    def _query(self, fn, ray_type, *args):
        try:
            check(fn(self.ctx.handle, self.handle, *args))
        except RegistryError:
            raise registry_error(self.custom_geom_types()[0] if self.custom_geom_types() else SPHERE_GEOM_TYPE,
                                 ray_type) from None

    def closest_hit_batch(self, origins, dirs, t_min, t_max, ray_mask, ray_type, registry, with_stats):
        self._bind(registry, ray_type)
        mask = _check_mask(ray_mask)
        origins = np.ascontiguousarray(origins, dtype=np.float64).reshape(-1, 3)
        dirs = np.ascontiguousarray(dirs, dtype=np.float64).reshape(-1, 3)
        n = origins.shape[0]
        if dirs.shape[0] != n:
            raise ValueError("origins and dirs must have the same length")
        tmin, tmin_s = t_range(t_min, n)
        tmax, tmax_s = t_range(t_max, n)
        t, u, v = host_empty(n, np.float64), host_empty(n, np.float64), host_empty(n, np.float64)
        inst, prim = host_empty(n, np.int64), host_empty(n, np.int64)
        nrm = host_empty((n, 3), np.float64)
        stats = host_empty((n, 2), np.int64) if with_stats else None
        self._query(lib().rt_tlas_closest_host, ray_type, n, ptr(origins), ptr(dirs), ptr(tmin), ptr(tmax), tmin_s,
                    tmax_s, mask, ptr(t), ptr(inst), ptr(prim), ptr(u), ptr(v), ptr(nrm), ptr(stats))
        res = (t, inst, prim, u, v, nrm)
        return res + (stats,) if with_stats else res

    def any_hit_batch(self, origins, dirs, t_min, t_max, ray_mask, ray_type, registry):
        self._bind(registry, ray_type)
        mask = _check_mask(ray_mask)
        origins = np.ascontiguousarray(origins, dtype=np.float64).reshape(-1, 3)
        dirs = np.ascontiguousarray(dirs, dtype=np.float64).reshape(-1, 3)
        n = origins.shape[0]
        if dirs.shape[0] != n:
            raise ValueError("origins and dirs must have the same length")
        tmin, tmin_s = t_range(t_min, n)
        tmax, tmax_s = t_range(t_max, n)
        out = host_empty(n, np.uint8)
        self._query(lib().rt_tlas_any_host, ray_type, n, ptr(origins), ptr(dirs), ptr(tmin), ptr(tmax), tmin_s,
                    tmax_s, mask, ptr(out))
        return out.view(bool)

    def __del__(self):
        try:
            if self.handle and _native._lib is not None:
                _native._lib.rt_tlas_destroy(self.handle)
        except Exception:
            pass


def build_tlas(instances, blases, quality="balanced") -> Tlas:
    """accel.py:552-553."""
    return Tlas(instances, blases, quality)


def transform_ray_to_local(origin, direction, inverse_matrix):
    """accel.py:349-359: world ray -> instance-local ray (direction keeps its length)."""
    inv = np.asarray(inverse_matrix, dtype=np.float64)
    return inv[:, :3] @ np.asarray(origin, np.float64) + inv[:, 3], inv[:, :3] @ np.asarray(direction, np.float64)
