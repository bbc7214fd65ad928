"""world_size-2/3 gloo tests of the multi-GPU split + exchange (CPU; the oracle stands in for
the GPU renderer, torch.distributed point-to-point for librt's NCCL band gather)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2603_00292_b200 import distributed as D

W, H, SPP = 24, 18, 6


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _oracle_render_fn(sc):
    def fn(accum, samples, bands):
        s0, s1 = samples
        out = np.zeros((H * W, 4))
        rays = 0
        if bands is None:
            _, rays = sc.render_frame(W, H, s1 - s0, "pt", max_depth=5, s0=s0, acc=out)
        else:
            stride, off = bands
            for r in range(off, (H + 3) // 4, stride):
                y0, y1 = 4 * r, min(4 * r + 4, H)
                _, rr = sc.render_frame(W, H, s1 - s0, "pt", max_depth=5, s0=s0, pix_lo=y0 * W, pix_hi=y1 * W,
                                        acc=out)
                rays += rr
        accum += torch.from_numpy(out.astype(np.float32))
        return rays
    return fn


def _worker(rank, world, port, mode, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle
        from paper_2603_00292_b200 import scenes
        sc = oracle.scene_from_description(scenes.cornell_description())
        acc = torch.zeros((H * W, 4), dtype=torch.float32)
        rays, acc = D.render_split(_oracle_render_fn(sc), acc, mode, SPP, width=W, height=H)
        if rank == 0:
            q.put((rays, acc.numpy().copy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("mode,world", [("samples", 2), ("tiles", 2), ("tiles", 3)])
def test_split_and_exchange(oracle_mod, mode, world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, mode, q)) for r in range(world)]
    for p in procs:
        p.start()
    rays, acc = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    from paper_2603_00292_b200 import scenes
    sc = oracle_mod.scene_from_description(scenes.cornell_description())
    full, full_rays = sc.render_frame(W, H, SPP, "pt", max_depth=5)
    assert rays == full_rays
    assert np.allclose(acc.reshape(H, W, 4), full, rtol=1e-5, atol=1e-5)
    assert np.all(acc[:, 3] == SPP)       # every pixel got every sample exactly once
    if mode == "tiles":                   # each pixel rendered on one rank: the 1-GPU values exactly
        assert np.array_equal(acc.reshape(H, W, 4), full.astype(np.float32))


def test_slices_and_bands_partition():
    for world in (1, 2, 3, 4, 8):
        cover = []
        for r in range(world):
            s0, s1 = D.sample_slice(r, world, 1024)
            cover.extend(range(s0, s1))
        assert cover == list(range(1024))
        rows = sorted(y for r in range(world) for y in D.band_rows(2160, r, world))
        assert rows == list(range(2160))
    with pytest.raises(ValueError):
        D.sample_slice(2, 2, 8)
