"""render_frame on the GPU (drop-in for integrators.py:426-473 of the reference).

Same signature and validation as the reference plus GPU knobs: ``kernel``
("mega" | "wavefront"; ao and pt-nee run in the megakernel) and ``samples``
(a [s0, s1) window of GLOBAL sample indices, for the sample split across
GPUs).  ``render_into`` accumulates into a caller-owned CUDA (H*W, 4) float32
tensor and keeps it on the device; ``resolve_device`` turns such a buffer
into display bytes on the GPU (scene_io.py:349-355).
"""

import warnings
from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import _native
from ._native import RenderParams, check, lib, ptr
from .scene_io import AccumBuffer

INTEGRATORS = ("eye", "ao", "pt", "pt-nee")
KERNELS = {"mega": _native.RT_KERNEL_MEGA, "wavefront": _native.RT_KERNEL_WAVEFRONT}


@dataclass
class IntegratorConfig:
    """integrators.py:56-74."""

    max_depth: int = 8
    sky_color: Optional[np.ndarray] = None
    ao_ray_count: int = 16
    ao_max_length: float = 1e30
    normal_offset: Optional[float] = None

    def __post_init__(self):
        if self.max_depth < 1:
            raise ValueError("max_depth must be >= 1")
        if self.ao_ray_count < 1:
            raise ValueError("ao_ray_count must be >= 1")
        if not (self.ao_max_length > 0.0):
            raise ValueError("ao_max_length must be > 0")
        if self.sky_color is not None:
            self.sky_color = np.asarray(self.sky_color, dtype=np.float64).reshape(3)
        if self.normal_offset is not None and not (self.normal_offset > 0.0):
            raise ValueError("normal_offset must be > 0")


def resolve_config(scene, cfg):
    """integrators.py:405-413."""
    cfg = IntegratorConfig() if cfg is None else cfg
    sky = cfg.sky_color if cfg.sky_color is not None else scene.sky
    off = cfg.normal_offset
    if off is None:
        diag = scene.diagonal()
        off = 1e-4 * diag if diag > 0.0 else 1e-4
    return cfg, np.asarray(sky, np.float64), float(off)


def make_params(scene, width, height, s0, s1, integrator, seed, cfg, jitter, kernel="mega", pix_lo=0, pix_hi=0):
    if integrator not in INTEGRATORS:
        raise ValueError(f"unknown integrator {integrator!r}, expected one of {INTEGRATORS}")
    if integrator == "pt-nee" and len(scene.lights) == 0:
        warnings.warn("scene has no emissive triangles, falling back to plain path tracing")
        integrator = "pt"
    if kernel not in KERNELS:
        raise ValueError(f"unknown kernel {kernel!r}, expected one of {tuple(KERNELS)}")
    if kernel == "wavefront" and integrator not in ("eye", "pt"):
        raise ValueError(f"integrator {integrator!r} runs in the megakernel only (kernel='mega')")
    if hasattr(scene, "sync_render"):
        scene.sync_render()          # two-level: re-flatten after refresh_instance_bounds
    cfg, sky, off = resolve_config(scene, cfg)
    scene.camera.validate_distortion()
    p = RenderParams()
    p.width, p.height, p.s0, p.s1 = int(width), int(height), int(s0), int(s1)
    p.seed = int(seed) & 0xFFFFFFFFFFFFFFFF
    p.jitter = 1 if jitter else 0
    p.integrator = {"eye": _native.RT_INTEG_EYE, "ao": _native.RT_INTEG_AO, "pt": _native.RT_INTEG_PT,
                    "pt-nee": _native.RT_INTEG_PTNEE}[integrator]
    p.max_depth = int(cfg.max_depth)
    p.ao_count = int(cfg.ao_ray_count)
    p.ao_length = float(min(cfg.ao_max_length, 3.0e38))
    p.kernel = KERNELS[kernel]
    for k, x in enumerate(scene.camera.as_tuple()):
        p.cam[k] = x
    for k in range(3):
        p.sky[k] = float(sky[k])
        p.background[k] = float(scene.background[k])
    p.normal_offset = off
    p.pix_lo, p.pix_hi = int(pix_lo), int(pix_hi)
    return p


def render_into(scene, accum, width, height, spp=1, integrator="pt", seed=0, cfg=None, jitter=True,
                kernel="mega", samples=None, pixels=None, count_rays=True, bands=None):
    """Device form: accumulate into a CUDA (H*W, 4) f32 tensor; returns the ray count (or None).

    samples: [s0, s1) global sample indices (sample split); pixels: row-major
    [lo, hi) pixel range; bands: (stride, offset) interleaved 4-row tile bands
    (tile split, whole-frame ranges only)."""
    s0, s1 = (0, spp) if samples is None else samples
    pix_lo, pix_hi = (0, 0) if pixels is None else pixels
    p = make_params(scene, width, height, s0, s1, integrator, seed, cfg, jitter, kernel, pix_lo, pix_hi)
    if bands is not None:
        p.band_stride, p.band_offset = int(bands[0]), int(bands[1])
    rays = np.zeros(1, np.uint64)
    flat = getattr(scene, "render_tlas", None) or scene.tlas   # two-level scenes render their device flatten
    check(lib().rt_render(flat.ctx.handle, flat.handle, p, ptr(accum), ptr(rays) if count_rays else None))
    return int(rays[0]) if count_rays else None


_PIPE_CHUNKS = 4                 # row chunks of a pipelined eye render_frame (rt_render_host)
_PIPE_MIN_PIXELS = 1 << 20


def render_frame(scene, width: int, height: int, spp: int, integrator: str = "pt", seed: int = 0,
                 workers: int = 1, cfg: Optional[IntegratorConfig] = None, jitter: bool = True,
                 return_stats: bool = False, kernel: str = "mega", samples=None, bands=None, gpus: int = 1):
    """Render a full frame into a fresh AccumBuffer (float64 host copy of the fp32 device sums).

    ``workers`` (the reference's CPU thread count, integrators.py:426-463) is accepted and
    validated; it cannot change the result (the reference's frames are bit-identical for any
    worker count, SPEC AC9) and the GPU needs no host threads, so it selects nothing here.
    ``gpus=N`` renders on GPUs [d, d+N) of the node, d = the scene's device: the scene is
    replicated (device-to-device clone of its built LBVH), GPU g renders the interleaved
    4-row tile bands r % N == g, and the bands are gathered into GPU d over NCCL
    (rt_multi_render).  Every pixel's samples are summed on one GPU, so the frame is
    bit-identical to ``gpus=1``.

    One native call (rt_render_host) renders and reads back: eye frames in the megakernel
    write their float64 rows directly (the exact widening of the fp32 sums), other frames
    are widened on the device; the rows reach pinned memory by DMA.  Large eye frames render
    in 4 row chunks so each chunk's readback overlaps the next chunk's render
    (return_stats=True renders in one launch to count rays).  `bands=(stride, offset)` renders only that GPU's interleaved
    4-row tile bands (the multi-GPU tile split); the other pixels stay 0.  The returned
    array lives in pinned host memory (PyTorch's caching host allocator) until freed."""
    import torch
    if width < 1 or height < 1 or spp < 1:
        raise ValueError("width, height, and spp must all be >= 1")
    if workers < 1:
        raise ValueError("workers must be >= 1")
    if gpus < 1:
        raise ValueError("gpus must be >= 1")
    if gpus > 1:
        return _render_frame_gpus(scene, width, height, spp, integrator, seed, cfg, jitter, return_stats, kernel,
                                  samples, gpus)
    if bands is not None and int(bands[0]) == 1:
        bands = None                                 # one GPU's "split" is the whole frame
    npix = height * width
    host = torch.empty((npix, 4), dtype=torch.float64, pin_memory=True)
    s0, s1 = (0, spp) if samples is None else samples
    p = make_params(scene, width, height, s0, s1, integrator, seed, cfg, jitter, kernel)
    if bands is not None:
        p.band_stride, p.band_offset = int(bands[0]), int(bands[1])
    # only primary-ray frames pipeline their readback: there it is comparable to the render;
    # a path-traced frame renders for far longer than its readback, and chunks add wave tails
    # (config 3 e2e 4849 -> 4164 Mrays/s when pipelined)
    nc = _PIPE_CHUNKS if integrator == "eye" and npix >= _PIPE_MIN_PIXELS and not return_stats else 1
    ray_count = np.zeros(1, np.uint64)
    flat = getattr(scene, "render_tlas", None) or scene.tlas
    check(lib().rt_render_host(flat.ctx.handle, flat.handle, p, ptr(host), nc,
                               ptr(ray_count) if return_stats else None))
    rays = int(ray_count[0]) if return_stats else None
    buf = AccumBuffer(width, height, host.numpy().reshape(height, width, 4))
    if return_stats:
        return buf, {"rays": rays}
    return buf


def _render_frame_gpus(scene, width, height, spp, integrator, seed, cfg, jitter, return_stats, kernel, samples,
                       gpus):
    """render_frame(gpus=N): tile split over N devices through rt_multi_render."""
    import torch
    from .distributed import render_frame_multi
    if samples is not None:
        raise ValueError("gpus > 1 renders whole sample ranges [0, spp)")
    dev0 = (getattr(scene, "render_tlas", None) or scene.tlas).ctx.device
    n_dev = torch.cuda.device_count()
    if dev0 + gpus > n_dev:
        raise ValueError(f"gpus={gpus} from device {dev0} needs {dev0 + gpus} devices, {n_dev} present")
    reps = [scene] + [scene.replica(dev0 + g) for g in range(1, gpus)]
    acc, rays = render_frame_multi(reps, width, height, spp, integrator, seed, cfg, jitter, kernel,
                                   return_device=True, mode="tiles")
    host = torch.empty((height * width, 4), dtype=torch.float64, pin_memory=True)
    host.copy_(acc.to(torch.float64), non_blocking=True)
    torch.cuda.current_stream(acc.device).synchronize()
    buf = AccumBuffer(width, height, host.numpy().reshape(height, width, 4))
    if return_stats:
        return buf, {"rays": rays}
    return buf


def resolve_device(ctx_or_scene, accum, width, height, gamma_encode=True) -> np.ndarray:
    """scene_io.py:349-355 on the GPU: (H*W, 4) f32 CUDA sums -> (H, W, 3) uint8 host image."""
    import torch
    ctx = ctx_or_scene.tlas.ctx if hasattr(ctx_or_scene, "tlas") else ctx_or_scene
    if accum.shape[0] != width * height:
        raise ValueError("accumulation buffer does not match the frame size")
    rgb = torch.empty((height * width * 3,), dtype=torch.uint8, device=accum.device)
    check(lib().rt_resolve(ctx.handle, ptr(accum), width * height, 1 if gamma_encode else 0, ptr(rgb)))
    return rgb.cpu().numpy().reshape(height, width, 3)


def raygen(scene, width, height, sample=0, seed=0, jitter=True):
    """Primary rays of one sample for every pixel, (W*H, 8) f32 on the device (parity helper)."""
    import torch
    p = make_params(scene, width, height, sample, sample + 1, "eye", seed, None, jitter)
    rays = torch.empty((width * height, 8), dtype=torch.float32, device=torch.device("cuda", scene.tlas.ctx.device))
    check(lib().rt_raygen(scene.tlas.ctx.handle, p, int(sample), ptr(rays)))
    scene.tlas.ctx.sync()
    return rays
