"""Multi-GPU work split and the single accumulation reduce.

One process per GPU (torch.distributed, NCCL over NVLink/NVSwitch on the B200
box; gloo in the CPU tests).  The scene and its LBVH are REPLICATED: every rank
builds the identical LBVH from the same triangles (the build is deterministic,
so replicas are bit-equal).  Two splits, both without any data-path
collective until the very end:

* sample split (path tracing, configs 3/5): rank g renders global sample
  indices [g*spp/G, (g+1)*spp/G) of every pixel.  The per-(seed, pixel,
  sample) stream hash uses the GLOBAL index (sampling.py:67-73), so the random
  numbers are exactly those of a 1-GPU run; only the fp32 summation order of
  the final reduce differs.
* tile split (primary rays, config 4): rank g renders the 4-row tile bands
  r with r % G == g (interleaved for load balance).  Untouched pixels stay 0,
  so the same sum-reduce assembles the frame.

Then exactly one ``reduce(sum, dst=0)`` of the (H*W, 4) fp32 accumulation
buffer (33.2 MB at 1080p).  ``render_fn`` is injectable so the collective
logic is tested with gloo and the CPU oracle (tests/test_distributed.py).
"""

import numpy as np


def sample_slice(rank: int, world: int, spp: int):
    """Global sample window [s0, s1) of one rank (contiguous, sizes differ by <= 1)."""
    if not (0 <= rank < world) or spp < 1:
        raise ValueError("bad rank / world / spp")
    return rank * spp // world, (rank + 1) * spp // world


def band_split(rank: int, world: int):
    """(stride, offset) of the interleaved 4-row tile bands of one rank."""
    if not (0 <= rank < world):
        raise ValueError("bad rank / world")
    return world, rank


def band_rows(height: int, rank: int, world: int):
    """Image rows a rank renders under band_split (host-side mirror of the kernel mapping)."""
    rows = []
    for r in range(rank, (height + 3) // 4, world):
        rows.extend(range(4 * r, min(4 * r + 4, height)))
    return rows


def render_split(render_fn, accum, mode, spp, group=None, dst=0):
    """Run this rank's share with render_fn, then one sum-reduce of ``accum`` to ``dst``.

    render_fn(accum, samples=(s0, s1) | None, bands=(stride, offset) | None) -> rays
    accum: torch tensor (H*W, 4) float32 on this rank's device (CPU for gloo).
    Returns (rays rendered by all ranks, reduced accum on dst / partial elsewhere).
    """
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    if mode == "samples":
        rays = render_fn(accum, samples=sample_slice(rank, world, spp), bands=None)
    elif mode == "tiles":
        rays = render_fn(accum, samples=(0, spp), bands=band_split(rank, world))
    else:
        raise ValueError(f"unknown split {mode!r}")
    if world > 1:
        dist.reduce(accum, dst=dst, op=dist.ReduceOp.SUM, group=group)
        r = torch.tensor([float(rays or 0)], dtype=torch.float64, device=accum.device)
        dist.all_reduce(r, group=group)
        rays = int(r.item())
    return rays, accum


def render_frame_distributed(scene, width, height, spp, integrator="pt", seed=0, cfg=None, jitter=True,
                             kernel="mega", mode="samples", group=None):
    """GPU render_frame across all ranks; rank 0 gets the AccumBuffer, others None."""
    import torch
    import torch.distributed as dist
    from .integrators import render_into
    from .scene_io import AccumBuffer
    dev = torch.device("cuda", scene.tlas.ctx.device)
    acc = torch.zeros((width * height, 4), dtype=torch.float32, device=dev)

    def fn(a, samples, bands):
        return render_into(scene, a, width, height, spp, integrator, seed, cfg, jitter, kernel,
                           samples=samples, bands=bands)

    rays, acc = render_split(fn, acc, mode, spp, group)
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    if rank != 0:
        return None, rays
    return AccumBuffer(width, height, acc.cpu().numpy().astype(np.float64).reshape(height, width, 4)), rays


def render_frame_multi(scenes, width, height, spp, integrator="pt", seed=0, cfg=None, jitter=True, kernel="mega",
                       return_device=False, mode="samples"):
    """One process, several GPUs: ``scenes[g]`` is the replica compiled on device g.

    ``rt_multi_render`` (csrc/multi.cu) enqueues every device's share concurrently --
    the sample split (global sample indices, so the random numbers are those of a
    1-GPU run) or the tile-band split -- then ONE grouped NCCL reduce of the fp32
    accumulation buffers into GPU 0.  Returns (accum on GPU 0, rays) with
    return_device, else (AccumBuffer, rays)."""
    import ctypes
    import torch
    from ._native import RT_SPLIT_SAMPLES, RT_SPLIT_TILES, check, lib
    from .integrators import make_params
    from .scene_io import AccumBuffer
    G = len(scenes)
    if G < 1:
        raise ValueError("need at least one scene replica")
    if width < 1 or height < 1 or spp < 1:
        raise ValueError("width, height, and spp must all be >= 1")
    if mode not in ("samples", "tiles"):
        raise ValueError(f"unknown split {mode!r}")
    flats = [getattr(sc, "render_tlas", None) or sc.tlas for sc in scenes]
    accs = [torch.zeros((width * height, 4), dtype=torch.float32, device=torch.device("cuda", f.ctx.device))
            for f in flats]
    p = make_params(scenes[0], width, height, 0, spp, integrator, seed, cfg, jitter, kernel)
    ctxs = (ctypes.c_void_p * G)(*[f.ctx.handle.value for f in flats])
    hs = (ctypes.c_void_p * G)(*[f.handle.value for f in flats])
    ptrs = (ctypes.c_void_p * G)(*[a.data_ptr() for a in accs])
    rays = np.zeros(1, np.uint64)
    check(lib().rt_multi_render(G, ctxs, hs, p, ptrs, RT_SPLIT_SAMPLES if mode == "samples" else RT_SPLIT_TILES,
                                rays.ctypes.data_as(ctypes.c_void_p)))
    acc = accs[0]
    if return_device:
        return acc, int(rays[0])
    return AccumBuffer(width, height, acc.cpu().numpy().astype(np.float64).reshape(height, width, 4)), int(rays[0])
