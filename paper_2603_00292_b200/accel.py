"""Closest-hit queries on the GPU (drop-in for accel.py:1128-1156 of the reference).

``closest_hit_batch`` keeps the reference signature, dtypes and conventions:
float64 / int64 host arrays in and out, misses flagged by t < 0 with
inst = prim = -1, u = v = -1 and a zero normal, the 32-bit mask check, a
``with_stats`` tuple of (triangle tests, node visits) per ray.  Custom
primitives have no GPU intersector yet, so a registry argument raises
``RegistryError`` instead of silently falling back to the CPU.

``trace_closest`` is the device-resident form used by the benchmark: rays and
hits are CUDA buffers (torch tensors), nothing crosses PCIe.
"""

import numpy as np

from ._native import RegistryError, check, lib, ptr

FULL_MASK = 0xFFFFFFFF
DEFAULT_MAX_T = 1e30


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
    if registry is not None:
        raise RegistryError("custom intersectors are not available on the GPU path")
    mask = _check_mask(ray_mask)
    origins = np.ascontiguousarray(origins, dtype=np.float64).reshape(-1, 3)
    dirs = np.ascontiguousarray(dirs, dtype=np.float64).reshape(-1, 3)
    n = origins.shape[0]
    if dirs.shape[0] != n:
        raise ValueError("origins and dirs must have the same length")
    tmin = np.ascontiguousarray(np.broadcast_to(np.asarray(t_min, dtype=np.float64), (n,)))
    tmax = np.ascontiguousarray(np.broadcast_to(np.asarray(t_max, dtype=np.float64), (n,)))
    t = np.empty(n)
    inst = np.empty(n, np.int64)
    prim = np.empty(n, np.int64)
    u = np.empty(n)
    v = np.empty(n)
    nrm = np.empty((n, 3))
    stats = np.empty((n, 2), np.int64) if with_stats else None
    check(lib().rt_closest_hit_host(tl.ctx.handle, tl.handle, n, ptr(origins), ptr(dirs), ptr(tmin), ptr(tmax),
                                    mask, ptr(t), ptr(inst), ptr(prim), ptr(u), ptr(v), ptr(nrm), ptr(stats)))
    res = (t, inst, prim, u, v, nrm)
    return res + (stats,) if with_stats else res


def any_hit_batch(tlas, origins, dirs, t_min=0.0, t_max=DEFAULT_MAX_T, ray_mask: int = FULL_MASK,
                  ray_type: int = 0, registry=None) -> np.ndarray:
    """accel.py:1159-1174: True iff some accepted intersection lies in [t_min, t_max]."""
    tl = _tlas_of(tlas)
    if registry is not None:
        raise RegistryError("custom intersectors are not available on the GPU path")
    mask = _check_mask(ray_mask)
    origins = np.ascontiguousarray(origins, dtype=np.float64).reshape(-1, 3)
    dirs = np.ascontiguousarray(dirs, dtype=np.float64).reshape(-1, 3)
    n = origins.shape[0]
    if dirs.shape[0] != n:
        raise ValueError("origins and dirs must have the same length")
    tmin = np.ascontiguousarray(np.broadcast_to(np.asarray(t_min, dtype=np.float64), (n,)))
    tmax = np.ascontiguousarray(np.broadcast_to(np.asarray(t_max, dtype=np.float64), (n,)))
    out = np.zeros(n, np.uint8)
    check(lib().rt_any_hit_host(tl.ctx.handle, tl.handle, n, ptr(origins), ptr(dirs), ptr(tmin), ptr(tmax), mask,
                                ptr(out)))
    return out.astype(bool)


def trace_any(tlas, rays, hit, ray_mask: int = FULL_MASK):
    """Device form: rays (n, 8) f32 CUDA tensor -> hit (n,) uint8 CUDA tensor."""
    tl = _tlas_of(tlas)
    check(lib().rt_trace_any(tl.ctx.handle, tl.handle, rays.shape[0], ptr(rays), ptr(hit), _check_mask(ray_mask)))


def trace_closest(tlas, rays, hits, ray_mask: int = FULL_MASK, stats=None):
    """Device form: rays (n, 8) f32 CUDA tensor [o, tmin, d, tmax] -> hits (n, 4) [t, id, u, v]."""
    tl = _tlas_of(tlas)
    n = rays.shape[0]
    check(lib().rt_trace_closest(tl.ctx.handle, tl.handle, n, ptr(rays), ptr(hits), _check_mask(ray_mask),
                                 ptr(stats)))
