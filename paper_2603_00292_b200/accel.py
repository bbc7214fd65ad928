"""Closest-hit queries on the GPU (drop-in for accel.py:1128-1156 of the reference).

``closest_hit_batch`` keeps the reference signature, dtypes and conventions:
float64 / int64 host arrays in and out, misses flagged by t < 0 with
inst = prim = -1, u = v = -1 and a zero normal, the 32-bit mask check, a
``with_stats`` tuple of (triangle tests, node visits) per ray.

Custom primitives keep the reference's registry contract (accel.py:366-423,
1002-1014): an ``IntersectorRegistry`` maps (geometry type, ray type) to an
intersection function and its data.  On the GPU the function is the builtin
``sphere_intersector`` (a float64 device kernel, traverse.cuh); a registry
entry with any other function raises ``RegistryError`` instead of running on
the CPU.  With no entry for the scene's spheres, a ray that reaches one raises
the reference's ``RegistryError`` message.

``trace_closest`` is the device-resident form used by the benchmark: rays and
hits are CUDA buffers (torch tensors), nothing crosses PCIe.
"""

import math

import numpy as np

from ._native import RegistryError, check, host_empty, lib, ptr, t_range

FULL_MASK = 0xFFFFFFFF
DEFAULT_MAX_T = 1e30
TRIANGLES = 0                 # accel.py:41-43
CUSTOM = 1
SPHERE_GEOM_TYPE = 0
RT_TRACE_NO_CUSTOM = 1        # include/rt_b200.h


def _sphere_hit(ox, oy, oz, dx, dy, dz, t_min, t_max, cx, cy, cz, r):
    """geometry.py:334-363, scalar float64 (the device kernel is sphere_hit_f64)."""
    lx, ly, lz = ox - cx, oy - cy, oz - cz
    a = dx * dx + dy * dy + dz * dz
    b = 2.0 * (lx * dx + ly * dy + lz * dz)
    c = lx * lx + ly * ly + lz * lz - r * r
    disc = b * b - 4.0 * a * c
    if disc < 0.0:
        return -1.0, 0.0, 0.0, 0.0
    sq = math.sqrt(disc)
    q = -0.5 * (b + math.copysign(sq, b))
    t0, t1 = (0.0, 0.0) if q == 0.0 else (q / a, c / q)
    if t0 > t1:
        t0, t1 = t1, t0
    t = t0
    if t < t_min or t > t_max:
        t = t1
        if t < t_min or t > t_max:
            return -1.0, 0.0, 0.0, 0.0
    px, py, pz = ox + dx * t, oy + dy * t, oz + dz * t
    return t, (px - cx) / r, (py - cy) / r, (pz - cz) / r


def sphere_intersector(data, prim, ox, oy, oz, dx, dy, dz, t_min, t_max):
    """The builtin custom intersector (accel.py:396-401): data rows are (cx, cy, cz, radius).

    Registering it selects the GPU sphere kernel; this scalar form exists for
    single-ray use and documentation and is never called by the batch path."""
    base = prim * 4
    return _sphere_hit(ox, oy, oz, dx, dy, dz, t_min, t_max, data[base], data[base + 1], data[base + 2],
                       data[base + 3])


def sphere_data(spheres) -> np.ndarray:
    """accel.py:403-408: flatten (center, radius) rows into intersector data."""
    arr = np.ascontiguousarray(spheres, dtype=np.float64).reshape(-1, 4)
    if np.any(arr[:, 3] <= 0.0):
        raise ValueError("sphere radius must be > 0")
    return arr.ravel().copy()


def sphere_aabbs(spheres) -> np.ndarray:
    """accel.py:411-416."""
    arr = np.asarray(spheres, dtype=np.float64).reshape(-1, 4)
    out = np.empty((arr.shape[0], 6))
    out[:, :3] = arr[:, :3] - arr[:, 3:4]
    out[:, 3:] = arr[:, :3] + arr[:, 3:4]
    return out


class IntersectorRegistry:
    """accel.py:366-392: function table keyed by (geometry type, ray type)."""

    def __init__(self):
        self._entries = {}

    def register(self, geom_type: int, ray_type: int, fn, data):
        data = np.ascontiguousarray(data, dtype=np.float64).ravel()
        self._entries[(int(geom_type), int(ray_type))] = (fn, data)

    def entry(self, geom_type: int, ray_type: int):
        return self._entries.get((int(geom_type), int(ray_type)))

    def resolve(self, geom_types, ray_type: int):
        present = sorted({int(g) for g in geom_types})
        size = (present[-1] + 1) if present else 0
        slots = np.full(size, -1, dtype=np.int64)
        table = []
        for g in present:
            e = self._entries.get((g, int(ray_type)))
            if e is not None:
                slots[g] = len(table)
                table.append(e)
        return tuple(table), slots


def make_sphere_registry(data, ray_types=(0,)) -> IntersectorRegistry:
    """accel.py:419-423."""
    reg = IntersectorRegistry()
    for rt in ray_types:
        reg.register(SPHERE_GEOM_TYPE, rt, sphere_intersector, data)
    return reg


def registry_error(geom_type, ray_type):
    """accel.py:1011-1014."""
    return RegistryError(f"no intersection function registered for geometry type {geom_type} "
                         f"and ray type {ray_type}")


def _trace_flags(tl, registry, ray_type):
    """accel.py:1002-1008 _dispatch_for, for the GPU: 0 = spheres intersected on the
    device, RT_TRACE_NO_CUSTOM = no entry (reaching a sphere raises)."""
    if not getattr(tl, "n_spheres", 0):
        return 0
    e = registry.entry(SPHERE_GEOM_TYPE, ray_type) if registry is not None else None
    if e is None:
        return RT_TRACE_NO_CUSTOM
    fn, data = e
    if fn is not sphere_intersector:
        raise RegistryError("only the builtin sphere_intersector runs on the GPU (no CPU fallback for custom "
                            "intersection functions)")
    rows = tl.sphere_rows[:, 12:16].ravel()
    if data.shape != rows.shape or not np.array_equal(data, rows):
        raise ValueError("registered sphere data differs from the scene's spheres")
    return 0


def _call(fn, ray_type, *args):
    try:
        check(fn(*args))
    except RegistryError:
        raise registry_error(SPHERE_GEOM_TYPE, ray_type) from None


def _tlas_of(obj):
    return obj.tlas if hasattr(obj, "tlas") else obj


def _check_mask(ray_mask):
    if not (0 <= ray_mask <= FULL_MASK):
        raise ValueError("ray mask must fit in 32 bits")
    return int(ray_mask)


def closest_hit_batch(tlas, origins, dirs, t_min=0.0, t_max=DEFAULT_MAX_T, ray_mask: int = FULL_MASK,
                      ray_type: int = 0, registry=None, with_stats: bool = False):
    """Array-of-rays closest hit: (t, inst, prim, u, v, normal[, stats])."""
    tl = _tlas_of(tlas)
    if getattr(tl, "two_level", False):
        return tl.closest_hit_batch(origins, dirs, t_min, t_max, ray_mask, ray_type, registry, with_stats)
    flags = _trace_flags(tl, registry, ray_type)
    mask = _check_mask(ray_mask)
    origins = np.ascontiguousarray(origins, dtype=np.float64).reshape(-1, 3)
    dirs = np.ascontiguousarray(dirs, dtype=np.float64).reshape(-1, 3)
    n = origins.shape[0]
    if dirs.shape[0] != n:
        raise ValueError("origins and dirs must have the same length")
    tmin, tmin_s = t_range(t_min, n)
    tmax, tmax_s = t_range(t_max, n)
    # outputs in pinned memory: the device->host copies are full-rate async DMA
    t = host_empty(n, np.float64)
    inst = host_empty(n, np.int64)
    prim = host_empty(n, np.int64)
    u = host_empty(n, np.float64)
    v = host_empty(n, np.float64)
    nrm = host_empty((n, 3), np.float64)
    stats = host_empty((n, 2), np.int64) if with_stats else None
    _call(lib().rt_closest_hit_host, ray_type, tl.ctx.handle, tl.handle, n, ptr(origins), ptr(dirs), ptr(tmin),
          ptr(tmax), tmin_s, tmax_s, mask, ptr(t), ptr(inst), ptr(prim), ptr(u), ptr(v), ptr(nrm), ptr(stats), flags)
    res = (t, inst, prim, u, v, nrm)
    return res + (stats,) if with_stats else res


def any_hit_batch(tlas, origins, dirs, t_min=0.0, t_max=DEFAULT_MAX_T, ray_mask: int = FULL_MASK,
                  ray_type: int = 0, registry=None) -> np.ndarray:
    """accel.py:1159-1174: True iff some accepted intersection lies in [t_min, t_max]."""
    tl = _tlas_of(tlas)
    if getattr(tl, "two_level", False):
        return tl.any_hit_batch(origins, dirs, t_min, t_max, ray_mask, ray_type, registry)
    flags = _trace_flags(tl, registry, ray_type)
    mask = _check_mask(ray_mask)
    origins = np.ascontiguousarray(origins, dtype=np.float64).reshape(-1, 3)
    dirs = np.ascontiguousarray(dirs, dtype=np.float64).reshape(-1, 3)
    n = origins.shape[0]
    if dirs.shape[0] != n:
        raise ValueError("origins and dirs must have the same length")
    tmin, tmin_s = t_range(t_min, n)
    tmax, tmax_s = t_range(t_max, n)
    out = host_empty(n, np.uint8)
    _call(lib().rt_any_hit_host, ray_type, tl.ctx.handle, tl.handle, n, ptr(origins), ptr(dirs), ptr(tmin),
          ptr(tmax), tmin_s, tmax_s, mask, ptr(out), flags)
    return out.view(bool)


def trace_any(tlas, rays, hit, ray_mask: int = FULL_MASK, ray_type: int = 0, registry=None):
    """Device form: rays (n, 8) f32 CUDA tensor -> hit (n,) uint8 CUDA tensor.  Scenes with
    spheres intersect them unless ``registry`` is given without a sphere entry."""
    tl = _tlas_of(tlas)
    flags = _trace_flags(tl, registry, ray_type) if registry is not None else 0
    _call(lib().rt_trace_any, ray_type, tl.ctx.handle, tl.handle, rays.shape[0], ptr(rays), ptr(hit),
          _check_mask(ray_mask), flags)


def trace_closest(tlas, rays, hits, ray_mask: int = FULL_MASK, stats=None, ray_type: int = 0, registry=None):
    """Device form: rays (n, 8) f32 CUDA tensor [o, tmin, d, tmax] -> hits (n, 4) [t, id, u, v]."""
    tl = _tlas_of(tlas)
    n = rays.shape[0]
    flags = _trace_flags(tl, registry, ray_type) if registry is not None else 0
    _call(lib().rt_trace_closest, ray_type, tl.ctx.handle, tl.handle, n, ptr(rays), ptr(hits), _check_mask(ray_mask),
          ptr(stats), flags)
