"""The multi-GPU split on the real CUDA kernels with one GPU: 2-3 processes share cuda:0, each
renders its share of the frame with the megakernel (tile bands: the eye frames take the
probe schedule on their band set; sample slices for path tracing), and the shares meet through
torch.distributed (gloo) on the host -- the same split and exchange logic as the NCCL data
plane (distributed.render_split), which needs one GPU per rank.  The tile split must equal a
one-process frame bit for bit, the sample split up to the reduce's summation order."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

W, H = 200, 120


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _render_fn(sc, integ, cfg):
    from paper_2603_00292_b200 import render_into

    def fn(accum, samples, bands):
        d = torch.zeros(accum.shape, dtype=torch.float32, device="cuda")
        rays = render_into(sc, d, W, H, samples[1] - samples[0], integ, cfg=cfg, samples=samples, bands=bands)
        accum += d.cpu()
        return rays
    return fn


def _worker(rank, world, port, mode, integ, spp, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2603_00292_b200 import IntegratorConfig, compile_scene, scenes
        from paper_2603_00292_b200 import distributed as D
        desc = scenes.cornell_description() if integ == "pt" else scenes.sphere_description(200, 400)
        sc = compile_scene(desc)
        acc = torch.zeros((H * W, 4), dtype=torch.float32)
        rays, acc = D.render_split(_render_fn(sc, integ, IntegratorConfig(max_depth=5)), acc, mode, spp, width=W,
                                   height=H)
        if rank == 0:
            q.put((rays, acc.numpy().copy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("mode,world,integ,spp", [("tiles", 2, "eye", 1), ("tiles", 3, "eye", 1),
                                                   ("tiles", 2, "pt", 16), ("samples", 2, "pt", 16)])
def test_split_on_cuda_kernels(native, mode, world, integ, spp):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, mode, integ, spp, q)) for r in range(world)]
    for p in procs:
        p.start()
    rays, acc = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    from paper_2603_00292_b200 import IntegratorConfig, compile_scene, render_into, scenes
    desc = scenes.cornell_description() if integ == "pt" else scenes.sphere_description(200, 400)
    sc = compile_scene(desc)
    full = torch.zeros((H * W, 4), dtype=torch.float32, device="cuda")
    full_rays = render_into(sc, full, W, H, spp, integ, cfg=IntegratorConfig(max_depth=5))
    full = full.cpu().numpy()
    assert rays == full_rays
    assert np.all(acc[:, 3] == spp)                 # every pixel got every sample exactly once
    if mode == "tiles":                             # each pixel rendered by one rank: identical
        assert np.array_equal(acc, full)
    else:
        assert np.allclose(acc, full, rtol=1e-5, atol=1e-5)
