"""ctypes binding of librt_b200.so (the C ABI in include/rt_b200.h).

The product path has no CPU fallback: if the shared library is missing or no
sm_100 device is present, every call raises.  ctypes releases the GIL during
each call, so one Python thread per GPU works like the reference's worker
threads (integrators.py:460-463).
"""

import ctypes
import os
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# RT_B200_LIB: an alternative build of the same library (tools/ variant sweeps only)
LIB_PATH = os.environ.get("RT_B200_LIB") or os.path.join(_HERE, "librt_b200.so")

RT_OK = 0
RT_EINVAL = -1
RT_ECUDA = -2
RT_EUNSUPPORTED = -3
RT_EDEPTH = -4
RT_ENOMEM = -5
RT_ESTATE = -6
RT_ENCCL = -7
RT_EBUILD = -8
RT_SPLIT_SAMPLES = 0
RT_SPLIT_TILES = 1

RT_INTEG_EYE = 0
RT_INTEG_AO = 1
RT_INTEG_PT = 2
RT_INTEG_PTNEE = 3
RT_KERNEL_MEGA = 0
RT_KERNEL_WAVEFRONT = 1

_lib = None
_lock = threading.Lock()


class BuildError(ValueError):
    """accel.py:51-52."""


class RegistryError(LookupError):
    """accel.py:55-56."""


class NativeError(RuntimeError):
    pass


class RenderParams(ctypes.Structure):
    _fields_ = [("width", ctypes.c_int32), ("height", ctypes.c_int32),
                ("s0", ctypes.c_int32), ("s1", ctypes.c_int32),
                ("seed", ctypes.c_uint64), ("jitter", ctypes.c_int32),
                ("integrator", ctypes.c_int32), ("max_depth", ctypes.c_int32),
                ("kernel", ctypes.c_int32), ("cam", ctypes.c_float * 13),
                ("sky", ctypes.c_float * 3), ("background", ctypes.c_float * 3),
                ("normal_offset", ctypes.c_float), ("pix_lo", ctypes.c_int64),
                ("pix_hi", ctypes.c_int64), ("band_stride", ctypes.c_int32), ("band_offset", ctypes.c_int32),
                ("ao_count", ctypes.c_int32), ("ao_length", ctypes.c_float)]


class InstanceSrc(ctypes.Structure):
    """rt_instance_src (include/rt_b200.h)."""
    _fields_ = [("mesh", ctypes.c_int32), ("material", ctypes.c_int32), ("mask", ctypes.c_uint32),
                ("reserved", ctypes.c_int32), ("matrix", ctypes.c_double * 12), ("inverse", ctypes.c_double * 12)]


class CustomSrc(ctypes.Structure):
    """rt_custom_src (include/rt_b200.h)."""
    _fields_ = [("box", ctypes.c_float * 9), ("material", ctypes.c_int32), ("mask", ctypes.c_uint32),
                ("row", ctypes.c_double * 16)]


def lib():
    """Load the CUDA library; raises if it was not built (no silent fallback)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() "
                              "(this package has no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        vp, i32, i64, u32, ci = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint32, ctypes.c_int
        f64 = ctypes.c_double
        L.rt_last_error.restype = ctypes.c_char_p
        L.rt_version.restype = ctypes.c_char_p
        sigs = {
            "rt_device_count": [vp],
            "rt_ctx_create": [ci, vp],
            "rt_ctx_set_stream": [vp, vp],
            "rt_ctx_sync": [vp],
            "rt_ctx_counters": [vp, vp],
            "rt_set_probe_budget": [i32, vp],
            "rt_probe_stats": [vp, vp],
            "rt_scene_create": [vp, i64, vp, vp, vp, vp, vp, vp, vp, vp, i32, vp],
            "rt_bvh_build": [vp, vp, ci, vp],
            "rt_bvh_build_profiled": [vp, vp, ci, vp],
            "rt_scene_set_vertices": [vp, vp, vp],
            "rt_bvh_info": [vp, vp, vp, vp, vp],
            "rt_bvh_download": [vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp],
            "rt_trace_closest": [vp, vp, i64, vp, vp, u32, vp, i32],
            "rt_closest_hit_host": [vp, vp, i64, vp, vp, vp, vp, f64, f64, u32, vp, vp, vp, vp, vp, vp, vp, i32],
            "rt_render": [vp, vp, ctypes.POINTER(RenderParams), vp, vp],
            "rt_render_host": [vp, vp, ctypes.POINTER(RenderParams), vp, i32, vp],
            "rt_trace_any": [vp, vp, i64, vp, vp, u32, i32],
            "rt_any_hit_host": [vp, vp, i64, vp, vp, vp, vp, f64, f64, u32, vp, i32],
            "rt_scene_set_lights": [vp, vp, i32, vp],
            "rt_scene_set_spheres": [vp, vp, i32, vp],
            "rt_raygen": [vp, ctypes.POINTER(RenderParams), i32, vp],
            "rt_resolve": [vp, vp, i64, i32, vp],
            "rt_multi_render": [i32, vp, vp, ctypes.POINTER(RenderParams), vp, i32, vp],
            "rt_scene_set_local_normals": [vp, vp, vp],
            "rt_scene_set_local_rows": [vp, vp, vp],
            "rt_scene_set_custom": [vp, vp, i32, i64],
            "rt_tlas_create": [vp, i32, vp, vp, vp, vp, vp],
            "rt_tlas_update": [vp, vp, vp, vp],
            "rt_tlas_set_custom_data": [vp, vp, i32, i64, vp],
            "rt_tlas_info": [vp, vp, vp, vp],
            "rt_tlas_flatten": [vp, vp, vp, vp, vp, vp, i32, i32, vp, vp, vp, vp, i32, vp],
            "rt_tlas_closest_host": [vp, vp, i64, vp, vp, vp, vp, f64, f64, u32, vp, vp, vp, vp, vp, vp, vp],
            "rt_tlas_any_host": [vp, vp, i64, vp, vp, vp, vp, f64, f64, u32, vp],
            "rt_mesh_create": [vp, i64, i64, vp, i32, vp, vp, i32, vp],
            "rt_scene_refit_mesh": [vp, vp, vp, i64, vp, i32],
            "rt_scene_update_normals": [vp, vp],
            "rt_scene_get_vertices": [vp, vp, vp],
            "rt_scene_set_normals64": [vp, vp, vp],
            "rt_scene_set_local_frames": [vp, vp, i32, vp, vp],
            "rt_mesh_upload": [vp, i64, vp, i64, vp, vp, vp],
            "rt_mesh_upload_async": [vp, i64, vp, i64, vp, vp],
            "rt_mesh_upload_finish": [vp, vp, vp],
            "rt_mesh_info": [vp, vp, vp, vp],
            "rt_scene_compile": [vp, i32, vp, i32, vp, i32, vp, vp, vp, i32, vp],
            "rt_scene_get_ids": [vp, vp, vp, vp, vp, vp],
            "rt_scene_get_geometry": [vp, vp, vp, vp, vp, vp],
            "rt_scene_clone": [vp, vp, vp, vp],
            "rt_stream_draws": [vp, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64, i32, vp],
            "rt_comm_unique_id": [vp],
            "rt_comm_create": [vp, i32, i32, vp, vp],
            "rt_comm_gather_bands": [vp, vp, vp, i32, i32],
            "rt_comm_reduce_accum": [vp, vp, vp, i64],
            "rt_bands_copy": [vp, vp, vp, i32, i32, i32, i32, i32, vp],
        }
        for name, args in sigs.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = ci
        L.rt_ctx_destroy.argtypes = [vp]
        L.rt_ctx_destroy.restype = None
        L.rt_scene_destroy.argtypes = [vp]
        L.rt_scene_destroy.restype = None
        L.rt_tlas_destroy.argtypes = [vp]
        L.rt_tlas_destroy.restype = None
        L.rt_mesh_destroy.argtypes = [vp]
        L.rt_mesh_destroy.restype = None
        L.rt_comm_destroy.argtypes = [vp]
        L.rt_comm_destroy.restype = None
        _lib = L
        return L


def check(rc):
    if rc == RT_OK:
        return
    msg = lib().rt_last_error().decode(errors="replace")
    if rc == RT_EINVAL:
        raise ValueError(msg)
    if rc in (RT_EDEPTH, RT_EBUILD):
        raise BuildError(msg)
    if rc == RT_EUNSUPPORTED:
        raise RegistryError(msg)
    if rc == RT_ENOMEM:
        raise MemoryError(msg)
    raise NativeError(f"librt_b200 error {rc}: {msg}")


def host_empty(shape, dtype):
    """Output array in PINNED host memory (PyTorch's caching host allocator reuses freed
    blocks), so device->host copies into it run as full-rate async DMA."""
    import torch
    tdt = {np.dtype(np.float64): torch.float64, np.dtype(np.int64): torch.int64,
           np.dtype(np.uint8): torch.uint8, np.dtype(np.float32): torch.float32,
           np.dtype(np.int32): torch.int32}[np.dtype(dtype)]
    if not torch.cuda.is_available():
        return np.empty(shape, dtype)
    return torch.empty(shape, dtype=tdt, pin_memory=True).numpy()


def host_pinned_copy(a):
    """A pinned copy of a host array (for callers that reuse inputs across calls)."""
    out = host_empty(a.shape, a.dtype)
    np.copyto(out, a)
    return out


def t_range(t, n):
    """(array pointer source or None, scalar) for a t_min / t_max argument: a scalar is
    broadcast on the device instead of materialising an (n,) host array."""
    a = np.asarray(t, dtype=np.float64)
    if a.ndim == 0:
        return None, float(a)
    return np.ascontiguousarray(np.broadcast_to(a, (n,))), 0.0


def ptr(x):
    """Raw pointer of a numpy array or torch tensor (None passes through)."""
    if x is None:
        return None
    if hasattr(x, "data_ptr"):
        return ctypes.c_void_p(x.data_ptr())
    return x.ctypes.data_as(ctypes.c_void_p)


class Context:
    """One rt_ctx per CUDA device (owns a stream, counters, staging)."""

    _cache = {}

    def __init__(self, device=0):
        self.device = int(device)
        h = ctypes.c_void_p()
        check(lib().rt_ctx_create(self.device, ctypes.byref(h)))
        self.handle = h
        # issue everything on torch's current stream of this device, so device
        # buffers allocated / consumed by torch are ordered with our kernels
        import torch
        self.set_stream(torch.cuda.current_stream(self.device).cuda_stream)

    @classmethod
    def get(cls, device=0):
        with _lock:
            c = cls._cache.get(int(device))
        if c is None:
            c = cls(device)
            with _lock:
                cls._cache[int(device)] = c
        return c

    def set_stream(self, stream_ptr):
        self.stream_ptr = int(stream_ptr or 0)
        check(lib().rt_ctx_set_stream(self.handle, ctypes.c_void_p(self.stream_ptr) if self.stream_ptr else None))

    def sync(self):
        check(lib().rt_ctx_sync(self.handle))

    def __del__(self):
        try:
            if getattr(self, "handle", None) and _lib is not None:
                _lib.rt_ctx_destroy(self.handle)
        except Exception:
            pass
