"""Multi-GPU work split and the single accumulation exchange.

One process per GPU (torch.distributed launches and rendezvous; gloo in the CPU tests).
The scene and its LBVH are REPLICATED: every rank builds the identical LBVH from the same
triangles (the build is deterministic, so replicas are bit-equal).  Two splits, both
without any data-path collective until the very end:

* sample split (path tracing, configs 3/5): rank g renders global sample indices
  [g*spp/G, (g+1)*spp/G) of every pixel.  The per-(seed, pixel, sample) stream hash uses
  the GLOBAL index (sampling.py:67-73), so the random numbers are exactly those of a 1-GPU
  run; only the fp32 summation order of the final reduce differs.  Exchange: ONE
  reduce(sum) of the (H*W, 4) fp32 accumulation buffer into rank 0 (33.2 MB at 1080p).
* tile split (primary rays, config 4): rank g renders the 4-row tile bands r with
  r % G == g (interleaved for load balance).  Exchange: a band gather -- each rank sends
  only its own rows to rank 0 ((G-1)/G of one frame arrives at rank 0 in total), which
  writes them into its frame.  Every pixel's samples are summed on one GPU, so the frame
  is bit-identical to a 1-GPU render.

The GPU data plane is librt_b200's NCCL (csrc/multi.cu: rt_comm_*): torch.distributed only
carries the communicator's unique id.  ``render_fn`` is injectable and CPU tensors take a
torch.distributed (gloo) transport with the same band index math, so the split and
exchange logic is tested without GPUs (tests/test_distributed.py).
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


class NcclComm:
    """librt_b200's NCCL communicator of this rank (rt_comm_create), on the device of ``ctx``.
    Rank 0 makes the unique id; torch.distributed broadcasts its bytes (rendezvous only)."""

    _cache = {}

    def __init__(self, ctx, group=None):
        import ctypes
        import torch.distributed as dist
        from ._native import check, lib
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        uid = np.zeros(128, np.uint8)
        if self.rank == 0:
            check(lib().rt_comm_unique_id(uid.ctypes.data_as(ctypes.c_void_p)))
        obj = [uid.tobytes()]
        src = dist.get_global_rank(group, 0) if group is not None else 0
        dist.broadcast_object_list(obj, src=src, group=group)
        uid = np.frombuffer(obj[0], np.uint8).copy()
        h = ctypes.c_void_p()
        check(lib().rt_comm_create(ctx.handle, self.world, self.rank, uid.ctypes.data_as(ctypes.c_void_p),
                                   ctypes.byref(h)))
        self.handle = h
        self.ctx = ctx

    @classmethod
    def get(cls, ctx, group=None):
        key = (ctx.device, id(group))
        if key not in cls._cache:
            cls._cache[key] = cls(ctx, group)
        return cls._cache[key]

    def gather_bands(self, accum, width, height):
        from ._native import check, lib, ptr
        check(lib().rt_comm_gather_bands(self.handle, self.ctx.handle, ptr(accum), width, height))

    def reduce(self, accum):
        from ._native import check, lib, ptr
        check(lib().rt_comm_reduce_accum(self.handle, self.ctx.handle, ptr(accum), accum.shape[0]))

    def __del__(self):
        try:
            from . import _native
            if getattr(self, "handle", None) and _native._lib is not None:
                _native._lib.rt_comm_destroy(self.handle)
        except Exception:
            pass


def _torch_gather_bands(accum, width, height, group=None):
    """The band gather with torch.distributed point-to-point (CPU tensors / gloo): the same
    rows move as in rt_comm_gather_bands (csrc/multi.cu)."""
    import torch.distributed as dist
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    frame = accum.view(height, width, 4)
    glob = (lambda r: dist.get_global_rank(group, r)) if group is not None else (lambda r: r)
    if rank == 0:
        for g in range(1, world):
            rows = band_rows(height, g, world)
            if rows:
                buf = frame.new_empty((len(rows), width, 4))
                dist.recv(buf, src=glob(g), group=group)
                frame[rows] = buf
    else:
        rows = band_rows(height, rank, world)
        if rows:
            dist.send(frame[rows].contiguous(), dst=glob(0), group=group)


def render_split(render_fn, accum, mode, spp, group=None, width=None, height=None):
    """Run this rank's share with render_fn, then the split's one exchange into rank 0.

    render_fn(accum, samples=(s0, s1) | None, bands=(stride, offset) | None) -> rays
    accum: torch tensor (H*W, 4) float32 on this rank's device (CPU for gloo); the tile
    split needs width / height.  Returns (rays rendered by all ranks, accum: the frame on
    rank 0, this rank's partial elsewhere).  CUDA buffers go through librt_b200's NCCL
    (NcclComm); CPU buffers through torch.distributed (tests)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    if mode == "samples":
        rays = render_fn(accum, samples=sample_slice(rank, world, spp), bands=None)
    elif mode == "tiles":
        if width is None or height is None:
            raise ValueError("the tile split needs the frame width and height")
        rays = render_fn(accum, samples=(0, spp), bands=band_split(rank, world))
    else:
        raise ValueError(f"unknown split {mode!r}")
    if world > 1:
        if accum.is_cuda:
            from ._native import Context
            comm = NcclComm.get(Context.get(accum.device.index), group)
            if mode == "tiles":
                comm.gather_bands(accum, width, height)
            else:
                comm.reduce(accum)
        elif mode == "tiles":
            _torch_gather_bands(accum, width, height, group)
        else:
            dist.reduce(accum, dst=0, op=dist.ReduceOp.SUM, group=group)
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

    rays, acc = render_split(fn, acc, mode, spp, group, width, height)
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    if rank != 0:
        return None, rays
    # widened on the device (exact), one DMA into pinned memory
    host = torch.empty((width * height, 4), dtype=torch.float64, pin_memory=True)
    host.copy_(acc.to(torch.float64), non_blocking=True)
    torch.cuda.current_stream(dev).synchronize()
    return AccumBuffer(width, height, host.numpy().reshape(height, width, 4)), rays


def render_frame_multi(scenes, width, height, spp, integrator="pt", seed=0, cfg=None, jitter=True, kernel="mega",
                       return_device=False, mode="samples"):
    """One process, several GPUs: ``scenes[g]`` is the replica compiled on device g.

    ``rt_multi_render`` (csrc/multi.cu) enqueues every device's share concurrently --
    the sample split (global sample indices, so the random numbers are those of a
    1-GPU run) or the tile-band split -- then the split's one exchange into GPU 0 (a
    reduce of the fp32 accumulation buffers, or the band gather).  Returns (accum on
    GPU 0, rays) with return_device, else (AccumBuffer, rays)."""
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
    for sc in scenes:
        if hasattr(sc, "sync_render"):
            sc.sync_render()
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
