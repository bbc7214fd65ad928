"""CLI (cli.py:18-101 drop-in) and device resolve.

CPU part: usage errors and exit codes, scene-file round trip.  GPU part: the
PPM bytes of the reference CLI (tests/golden/cli_ppm.npz, produced by running
the reference's own ``pathtrace.cli.run`` on the same scene files) --
byte-exact for ``eye``; for the sampled integrators the fp32 frame matches
within the render tolerance, so bytes may differ by one level where the
float64 mean sits on a rounding boundary.
"""

import os

import numpy as np
import pytest

from paper_2603_00292_b200 import cli, scenes
from paper_2603_00292_b200.frames import frame_to_matrix
from paper_2603_00292_b200.scene_io import AccumBuffer, load_scene, resolve, write_scene_files
from rt_helpers import golden

JOBS = {
    "cornell_eye": ("cornell", ["--width", "64", "--height", "48", "--spp", "2", "--integrator", "eye"]),
    "cornell_pt": ("cornell", ["--width", "32", "--height", "24", "--spp", "4", "--integrator", "pt",
                               "--max-depth", "5"]),
    "cornell_ao": ("cornell", ["--width", "24", "--height", "16", "--spp", "2", "--integrator", "ao",
                               "--ao-rays", "4", "--no-gamma"]),
    "spheres_eye": ("spheres", ["--width", "48", "--height", "36", "--spp", "1", "--integrator", "eye"]),
    "spheres_nee": ("spheres", ["--width", "24", "--height", "18", "--spp", "2", "--integrator", "pt-nee",
                                "--max-depth", "4", "--seed", "3"]),
}


def test_usage_errors_exit_2(capsys):
    assert cli.run([]) == 2                                    # --scene/--out required
    assert cli.run(["--scene", "x", "--out", "y", "--integrator", "bogus"]) == 2
    assert cli.run(["--scene", "x", "--out", "y", "--device", "cpu"]) == 2   # no CPU device


def test_runtime_errors_exit_1(tmp_path, capsys):
    assert cli.run(["--scene", str(tmp_path / "missing.scn"), "--out", str(tmp_path / "o.ppm")]) == 1
    assert "pathtrace: error:" in capsys.readouterr().err
    assert not os.path.exists(tmp_path / "o.ppm")


@pytest.mark.parametrize("make", [scenes.cornell_description, scenes.spheres_description])
def test_scene_files_round_trip(tmp_path, make):
    d = make()
    e = load_scene(write_scene_files(d, str(tmp_path)))
    for k in d.meshes:
        assert np.array_equal(d.meshes[k].vertices, e.meshes[k].vertices)
        assert np.array_equal(d.meshes[k].faces, e.meshes[k].faces)
    for a, b in zip(d.instances + d.spheres, e.instances + e.spheres):
        assert np.array_equal(frame_to_matrix(a.frame), frame_to_matrix(b.frame))
        assert a.mask == b.mask and a.material == b.material
    for k in d.materials:
        assert np.array_equal(d.materials[k].color, e.materials[k].color)
    assert np.array_equal(d.sky, e.sky) and np.array_equal(d.background, e.background)


def _scene_paths(tmp_path):
    return {"cornell": write_scene_files(scenes.cornell_description(), str(tmp_path / "c")),
            "spheres": write_scene_files(scenes.spheres_description(), str(tmp_path / "s"))}


@pytest.mark.gpu
@pytest.mark.parametrize("name", list(JOBS))
def test_cli_ppm_vs_reference(native, tmp_path, name, capsys):
    g = golden("cli_ppm")
    scn, args = JOBS[name]
    out = tmp_path / (name + ".ppm")
    assert cli.run(["--scene", _scene_paths(tmp_path)[scn], "--out", str(out)] + args) == 0
    assert "GPU" in capsys.readouterr().err
    got = np.frombuffer(out.read_bytes(), dtype=np.uint8)
    ref = g[name]
    assert got.shape == ref.shape
    hdr = ref.tobytes().index(b"255\n") + 4
    assert got[:hdr].tobytes() == ref[:hdr].tobytes()
    diff = np.abs(got[hdr:].astype(int) - ref[hdr:].astype(int))
    if name.endswith("_eye"):
        assert diff.max() == 0
    else:
        assert diff.max() <= 1 and np.mean(diff > 0) <= 0.01, (diff.max(), np.mean(diff > 0))


@pytest.mark.gpu
def test_cli_stdout_and_gpus_auto(native, tmp_path, capfd):
    scn = _scene_paths(tmp_path)["cornell"]
    assert cli.run(["--scene", scn, "--out", "-", "--width", "8", "--height", "4", "--spp", "1",
                    "--gpus", "auto", "--integrator", "eye"]) == 0
    out = capfd.readouterr().out
    assert out.startswith("P6\n8 4\n255\n")


@pytest.mark.gpu
def test_resolve_device_matches_host(native):
    import torch
    from paper_2603_00292_b200 import compile_scene, render_into
    from paper_2603_00292_b200.integrators import resolve_device
    sc = compile_scene(scenes.cornell_description())
    acc = torch.zeros((40 * 30, 4), dtype=torch.float32, device="cuda")
    render_into(sc, acc, 40, 30, 3, "pt")
    host = AccumBuffer(40, 30, acc.cpu().numpy().astype(np.float64).reshape(30, 40, 4))
    for gamma in (True, False):
        assert np.array_equal(resolve_device(sc, acc, 40, 30, gamma), resolve(host, gamma))
    with pytest.raises(ValueError, match="zero samples"):
        resolve_device(sc, torch.zeros((4, 4), device="cuda"), 2, 2)


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["samples", "tiles"])
def test_multi_render_native(native, mode):
    """rt_multi_render (the --gpus path) on the devices present: the split frame equals
    the single-device frame (one device: bit-identical; more: fp32 reduce order only)."""
    import torch
    from paper_2603_00292_b200 import IntegratorConfig, compile_scene, render_frame
    from paper_2603_00292_b200.distributed import render_frame_multi
    desc = scenes.cornell_description()
    n = torch.cuda.device_count()
    reps = [compile_scene(desc, device=g) for g in range(n)]
    cfg = IntegratorConfig(max_depth=5)
    spp = 6 if mode == "samples" else 1
    integ = "pt" if mode == "samples" else "eye"
    acc2, rays2 = render_frame_multi(reps, 40, 30, spp, integ, cfg=cfg, mode=mode)
    acc1, st = render_frame(reps[0], 40, 30, spp, integ, cfg=cfg, return_stats=True)
    assert rays2 == st["rays"]
    assert np.array_equal(acc2.data[:, :, 3], acc1.data[:, :, 3])
    if n == 1:
        assert np.array_equal(acc2.data, acc1.data)
    else:
        assert np.allclose(acc2.data, acc1.data, rtol=1e-5, atol=1e-5)
    with pytest.raises(ValueError, match="distinct device"):
        render_frame_multi([reps[0], reps[0]], 8, 8, 2, "pt", cfg=cfg)


@pytest.mark.gpu
def test_multi_render_nccl_plumbing(native):
    """The dlopen'ed NCCL reduce path of rt_multi_render, forced on one device."""
    import subprocess
    import sys
    code = ("import numpy as np; from paper_2603_00292_b200 import compile_scene, render_frame, scenes; "
            "from paper_2603_00292_b200.distributed import render_frame_multi; "
            "sc = compile_scene(scenes.cornell_description()); "
            "a, r = render_frame_multi([sc], 16, 12, 4, 'pt'); b = render_frame(sc, 16, 12, 4, 'pt'); "
            "assert np.array_equal(a.data, b.data); print('nccl ok', r)")
    env = dict(os.environ, RT_MULTI_FORCE_NCCL="1")
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env,
                         cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))), timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    assert "nccl ok" in out.stdout
