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
def test_render_frame_multi_replicas_sum(native):
    """--gpus N logic on one device: two replicas split the samples, partial sums add up
    to the single-replica frame (fp32 addition order differs only at rounding level)."""
    from paper_2603_00292_b200 import IntegratorConfig, compile_scene, render_frame
    from paper_2603_00292_b200.distributed import render_frame_multi
    desc = scenes.cornell_description()
    reps = [compile_scene(desc), compile_scene(desc)]
    cfg = IntegratorConfig(max_depth=5)
    acc2, rays2 = render_frame_multi(reps, 40, 30, 6, "pt", cfg=cfg)
    acc1, st = render_frame(reps[0], 40, 30, 6, "pt", cfg=cfg, return_stats=True)
    assert rays2 == st["rays"]
    assert np.array_equal(acc2.data[:, :, 3], acc1.data[:, :, 3])
    assert np.allclose(acc2.data, acc1.data, rtol=1e-5, atol=1e-5)
