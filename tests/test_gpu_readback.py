"""render_frame's native readback (rt_render_host, csrc/render.cu).

Eye frames in the megakernel write float64 rows themselves (optionally in row chunks whose
copies overlap the next chunk's render); every other frame renders into fp32 sums widened on
the device.  Either way the host array must be the exact float64 widening of what rt_render
accumulates into zeroed fp32 sums -- for any chunk count, ragged frames, several samples,
sample windows and tile-band shares (other pixels 0), and after a larger frame has left
stale rows in the scratch."""

import ctypes

import numpy as np
import pytest
import torch

from paper_2603_00292_b200 import IntegratorConfig, _native, compile_scene, render_frame, render_into, scenes
from paper_2603_00292_b200.integrators import make_params

pytestmark = pytest.mark.gpu


def device_frame(sc, w, h, spp, integ, samples=None, bands=None, cfg=None, kernel="mega"):
    acc = torch.zeros((h * w, 4), dtype=torch.float32, device="cuda")
    rays = render_into(sc, acc, w, h, spp, integ, cfg=cfg, samples=samples, bands=bands, kernel=kernel)
    return acc.cpu().numpy().astype(np.float64), rays


def host_frame(sc, w, h, spp, integ, n_chunks, samples=None, bands=None, cfg=None, kernel="mega", count=True):
    s0, s1 = (0, spp) if samples is None else samples
    p = make_params(sc, w, h, s0, s1, integ, 0, cfg, True, kernel)
    if bands is not None:
        p.band_stride, p.band_offset = bands
    out = torch.full((h * w, 4), -1.0, dtype=torch.float64, pin_memory=True)
    rays = np.zeros(1, np.uint64)
    _native.check(_native.lib().rt_render_host(sc.tlas.ctx.handle, sc.tlas.handle, p, _native.ptr(out), n_chunks,
                                               rays.ctypes.data_as(ctypes.c_void_p) if count else None))
    return out.numpy().copy(), int(rays[0])


@pytest.fixture(scope="module")
def sphere(native):
    return compile_scene(scenes.sphere_description())


@pytest.mark.parametrize("w,h,spp,nc", [(1920, 1080, 1, 4), (1920, 1080, 1, 8), (1920, 1080, 2, 3),
                                        (1001, 603, 1, 4), (37, 5, 1, 4), (8, 4, 1, 2), (640, 360, 1, 1)])
def test_eye_readback_exact(sphere, w, h, spp, nc):
    ref, rays = device_frame(sphere, w, h, spp, "eye")
    got, grays = host_frame(sphere, w, h, spp, "eye", nc)            # counted: one launch
    assert np.array_equal(got, ref)
    assert grays == rays
    got, _ = host_frame(sphere, w, h, spp, "eye", nc, count=False)   # chunked when it can be
    assert np.array_equal(got, ref)


def test_eye_partial_frames_and_shares_exact(sphere):
    w, h = 1920, 1080
    host_frame(sphere, 2400, 1200, 1, "eye", 4)                    # stale rows in the scratch
    for kw in ({"samples": (3, 5)}, {"bands": (3, 1)}, {"bands": (2, 0)}):
        ref, rays = device_frame(sphere, w, h, 1, "eye", **kw)
        for nc in (1, 4):
            got, _ = host_frame(sphere, w, h, 1, "eye", nc, count=False, **kw)
            assert np.array_equal(got, ref), (kw, nc)


@pytest.mark.parametrize("kernel", ["mega", "wavefront"])
def test_pt_readback_exact(native, kernel):
    sc = compile_scene(scenes.cornell_description())
    cfg = IntegratorConfig(max_depth=5)
    ref, rays = device_frame(sc, 320, 240, 12, "pt", cfg=cfg, kernel=kernel)
    got, grays = host_frame(sc, 320, 240, 12, "pt", 4, cfg=cfg, kernel=kernel)   # widened on the device
    assert np.array_equal(got, ref)
    assert grays == rays
    ref, _ = device_frame(sc, 320, 240, 4, "eye", kernel="wavefront")
    got, _ = host_frame(sc, 320, 240, 4, "eye", 4, kernel="wavefront")
    assert np.array_equal(got, ref)


def test_render_frame_matches_device_frame(sphere):
    ref, rays = device_frame(sphere, 1920, 1080, 1, "eye")
    buf = render_frame(sphere, 1920, 1080, 1, "eye")
    assert np.array_equal(buf.data.reshape(-1, 4), ref)
    buf, st = render_frame(sphere, 1920, 1080, 1, "eye", return_stats=True)
    assert np.array_equal(buf.data.reshape(-1, 4), ref)
    assert st["rays"] == rays


def test_bad_chunk_count(sphere):
    p = make_params(sphere, 64, 64, 0, 1, "eye", 0, None, True, "mega")
    out = np.zeros((64 * 64, 4))
    assert _native.lib().rt_render_host(sphere.tlas.ctx.handle, sphere.tlas.handle, p, _native.ptr(out), 0,
                                        None) != 0
