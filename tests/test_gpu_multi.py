"""Multi-GPU pieces on the GPU.

On a 1-GPU box: the render replica (rt_scene_clone) renders and downloads exactly like its
source, and the band gather's pack / unpack (rt_bands_copy, the kernels rt_comm_gather_bands
and rt_multi_render's tile split run around ncclSend / ncclRecv) reassemble a frame from
per-rank band renders bit for bit.  With >= 2 GPUs: render_frame(gpus=N) and rt_multi_render
against one GPU (skipped when fewer devices are present).
"""

import ctypes
import dataclasses

import numpy as np
import pytest
import torch

from paper_2603_00292_b200 import IntegratorConfig, compile_scene, render_frame, render_into, scenes
from paper_2603_00292_b200 import distributed as D
from paper_2603_00292_b200._native import check, lib, ptr

pytestmark = pytest.mark.gpu


def test_clone_renders_like_source(native):
    sc = compile_scene(scenes.cornell_description())
    rep = dataclasses.replace(sc, tlas=sc.tlas.clone(0), _replicas=None)
    for integ, spp in (("eye", 1), ("pt", 3)):
        a = render_frame(sc, 64, 48, spp, integ, seed=7, cfg=IntegratorConfig(max_depth=5))
        b = render_frame(rep, 64, 48, spp, integ, seed=7, cfg=IntegratorConfig(max_depth=5))
        assert np.array_equal(a.data, b.data)
    da, db = sc.tlas.download(), rep.tlas.download()
    for k in da:
        assert np.array_equal(da[k], db[k]), k


@pytest.mark.parametrize("G,W,H", [(2, 64, 48), (3, 40, 37), (4, 1920, 1080), (8, 96, 30)])
def test_band_gather_reassembles_frame(native, G, W, H):
    sc = compile_scene(scenes.cornell_description())
    cfg = IntegratorConfig(max_depth=5)
    full = torch.zeros((H * W, 4), dtype=torch.float32, device="cuda")
    render_into(sc, full, W, H, 2, "pt", seed=1, cfg=cfg)
    frame = torch.zeros_like(full)
    ctx = sc.tlas.ctx
    total_rows = 0
    for g in range(G):
        part = torch.zeros_like(full)
        render_into(sc, part, W, H, 2, "pt", seed=1, cfg=cfg, bands=D.band_split(g, G))
        rows = len(D.band_rows(H, g, G))
        compact = torch.full((max(rows, 1) * W, 4), -1.0, dtype=torch.float32, device="cuda")
        n = np.zeros(1, np.int64)
        check(lib().rt_bands_copy(ctx.handle, ptr(part), ptr(compact), W, H, g, G, 0, ptr(n)))
        assert n[0] == rows
        if rows:
            # the compact rows are exactly rank g's rows of its band render
            assert torch.equal(compact[: rows * W].view(rows, W, 4), part.view(H, W, 4)[D.band_rows(H, g, G)])
        check(lib().rt_bands_copy(ctx.handle, ptr(frame), ptr(compact), W, H, g, G, 1, ptr(n)))
        total_rows += rows
    torch.cuda.synchronize()
    assert total_rows == H
    assert torch.equal(frame, full)


def _two_gpus():
    if torch.cuda.device_count() < 2:
        pytest.skip("needs >= 2 GPUs")


@pytest.mark.parametrize("integ", ["eye", "pt"])
def test_render_frame_gpus_equals_one_gpu(native, integ):
    _two_gpus()
    n = min(torch.cuda.device_count(), 4)
    sc = compile_scene(scenes.cornell_description())
    one = render_frame(sc, 200, 120, 4, integ, seed=3, cfg=IntegratorConfig(max_depth=5))
    many = render_frame(sc, 200, 120, 4, integ, seed=3, cfg=IntegratorConfig(max_depth=5), gpus=n)
    assert np.array_equal(one.data, many.data)


def test_multi_render_sample_split(native):
    _two_gpus()
    n = min(torch.cuda.device_count(), 4)
    desc = scenes.cornell_description()
    reps = [compile_scene(desc, device=d) for d in range(n)]
    cfg = IntegratorConfig(max_depth=5)
    acc, rays = D.render_frame_multi(reps, 96, 64, 8, "pt", seed=2, cfg=cfg, return_device=True, mode="samples")
    one = torch.zeros((96 * 64, 4), dtype=torch.float32, device="cuda:0")
    r1 = render_into(reps[0], one, 96, 64, 8, "pt", seed=2, cfg=cfg)
    assert rays == r1
    assert torch.allclose(acc.cpu(), one.cpu(), rtol=1e-5, atol=1e-5)


def test_comm_single_rank_roundtrip(native):
    """librt's one-process-per-GPU communicator (rt_comm_*) end to end with one rank: unique
    id through torch.distributed (gloo), ncclCommInitRank, the reduce (identity for one
    rank) and the band gather (a no-op) on a rendered frame."""
    import os
    import socket
    import torch.distributed as dist
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=0, world_size=1)
    try:
        sc = compile_scene(scenes.cornell_description())
        acc = torch.zeros((64 * 48, 4), dtype=torch.float32, device="cuda")
        rays, acc = D.render_split(lambda a, samples, bands: render_into(sc, a, 64, 48, 2, "pt", seed=4,
                                                                          samples=samples, bands=bands),
                                   acc, "samples", 2)
        ref = torch.zeros_like(acc)
        render_into(sc, ref, 64, 48, 2, "pt", seed=4)
        comm = D.NcclComm.get(sc.tlas.ctx)
        comm.reduce(acc)
        comm.gather_bands(acc, 64, 48)
        torch.cuda.synchronize()
        assert torch.equal(acc, ref)
    finally:
        dist.destroy_process_group()
