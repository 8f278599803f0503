"""The reference's CALLERS of the hot path, reference vs GPU:
render_scene / fit_scene (src/fit3d.cpp:29-203) and fit_image (src/fit2d.cpp:45-188) of the C++
mirror (paper_2501_12369_b200/host/darbs_b200_fit.hpp, driven by host/fit_tool.cpp) on the
reference's own data files proj/data/demo_scene.txt + demo_cameras.txt, against what the
reference's own sources produced from the same files (tests/golden/fit.npz and tests/golden/fit/,
written by tests/golden/make_golden.py through oracle/_ref).

Bars:
  * render: every view within 2e-5 of the reference's render (the forward's image tolerance);
  * fit_scene, 50 iterations from the stored start on the stored float32 targets: the loss, L1 and
    D-SSIM curves within 1e-3 relative of the reference's over the first 25 iterations and within
    5e-3 through all 50 (measured: <= 1e-3 everywhere for four families; the sharply truncated
    inverse multiquadric, whose footprint is discontinuous at the cutoff, reaches 3e-3 by
    iteration 43 — FP32 parameters put a few pixels on the other side of a cutoff), PSNR curve
    and final PSNR within 0.1 dB, fitted primitives within 1e-3 of the parameter scale;
  * acceptance criterion 7 (tests/acceptance.cpp:419-470): 2000 iterations of self-reconstruction
    per kernel — Gaussian min-view PSNR >= 35 dB, every other family within 2 dB of the bar; the
    reference's own figures are printed beside ours (a 2000-step Adam trajectory in FP32 does not
    retrace an FP64 one, so these are thresholds, as in the reference);
  * acceptance criterion 8 (:474-521): a seeded rerun of render, fit-scene (25 iterations) and
    fit-image (n = 40, 60 iterations, seed 5) is byte-identical in the deterministic mode;
  * fit_image, 60 iterations: curves within 1e-3 relative, final PSNR within 0.1 dB.
"""
import os
import subprocess

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HOST = os.path.join(ROOT, "paper_2501_12369_b200", "host")
FIT = os.path.join(ROOT, "tests", "golden", "fit")
TOOL = os.path.join(HOST, "fit_tool")
KERNELS = ["gaussian", "half-cosine-sq", "raised-cosine", "mod-sinc", "inv-multiquadratic"]


@pytest.fixture(scope="module")
def tool():
    r = subprocess.run(["make", "-C", HOST, "fit_tool"], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    return TOOL


@pytest.fixture(scope="module")
def gold():
    return np.load(os.path.join(ROOT, "tests", "golden", "fit.npz"))


def run(tool, *args, timeout=600):
    r = subprocess.run([tool, *[str(a) for a in args]], capture_output=True, text=True, timeout=timeout)
    assert r.returncode == 0, r.stdout + r.stderr
    return r


def read_dsfl(path):
    raw = open(path, "rb").read()
    assert raw[:4] == b"DSFL"
    w, h, c = np.frombuffer(raw[4:16], dtype="<u4")
    return np.frombuffer(raw[16:], dtype="<f4").reshape(h, w, c).astype(np.float64)


def read_report(path):
    curve, views, rows, final = [], [], [], None
    for line in open(path):
        f = line.split()
        if f[0] == "curve":
            curve.append([float(x) for x in f[2:]])
        elif f[0] == "final":
            final = np.array([float(x) for x in f[1:]])
        elif f[0] == "view":
            views.append(float(f[2]))
        else:
            rows.append([float(x) for x in f[1:]])
    c = np.array(curve)
    return dict(loss=c[:, 0], l1=c[:, 1], dssim=c[:, 2], psnr=c[:, 3], final=final, per_view_psnr=np.array(views),
                rows=np.array(rows))


@pytest.mark.parametrize("name", KERNELS)
def test_render_scene_matches_the_reference(tool, gold, tmp_path, name):
    """`render` (tools/main.cpp:336-351): the four demo cameras."""
    run(tool, "render", os.path.join(FIT, "scene.txt"), os.path.join(FIT, "cameras.txt"), name, "default", tmp_path)
    ref = gold[f"{name}/render"]
    for v in range(ref.shape[0]):
        img = read_dsfl(tmp_path / f"view_{v}.dsfl")
        assert img.shape == ref[v].shape
        assert np.abs(img - ref[v]).max() <= 2e-5, (name, v, np.abs(img - ref[v]).max())


@pytest.mark.parametrize("name", KERNELS)
def test_fit_scene_tracks_the_reference_trajectory(tool, gold, tmp_path, name):
    out = tmp_path / "fit.txt"
    run(tool, "fit-scene", os.path.join(FIT, f"targets_{name}"), os.path.join(FIT, "cameras.txt"),
        os.path.join(FIT, "init_0.02.txt"), name, "default", 50, out)
    got = read_report(out)
    for key in ("loss", "l1", "dssim"):
        ref = gold[f"{name}/fit50/{key}"]
        rel = np.abs(got[key] - ref) / np.abs(ref)
        assert rel[:25].max() <= 1e-3, (name, key, int(rel[:25].argmax()), rel[:25].max())
        assert rel.max() <= 5e-3, (name, key, int(rel.argmax()), rel.max())
    assert np.abs(got["psnr"] - gold[f"{name}/fit50/psnr"]).max() <= 0.1
    assert abs(got["final"][1] - gold[f"{name}/fit50/final"][1]) <= 0.1
    assert np.abs(got["per_view_psnr"] - gold[f"{name}/fit50/per_view_psnr"]).max() <= 0.1
    prims = gold[f"{name}/fit50/primitives"]
    q = got["rows"].copy()
    # the mirror returns the normalised quaternion's realisation as the reference does (fit3d.cpp:17-25)
    assert np.abs(q - prims).max() <= 1e-3 * max(1.0, np.abs(prims).max()), np.abs(q - prims).max()


def test_acceptance_criterion_7_self_reconstruction(tool, gold, tmp_path):
    """tests/acceptance.cpp:419-470 through the GPU path: 2000 iterations per family."""
    finals, min_view = {}, {}
    for name in KERNELS:
        out = tmp_path / f"{name}.txt"
        run(tool, "fit-scene", os.path.join(FIT, "scene.txt"), os.path.join(FIT, "cameras.txt"),
            os.path.join(FIT, "init_0.02.txt"), name, "default", 2000, out, timeout=1200)
        got = read_report(out)
        finals[name], min_view[name] = got["final"][1], got["per_view_psnr"].min()
        print(f"{name}: GPU {finals[name]:.2f} dB (min view {min_view[name]:.2f}); reference "
              f"{gold[name + '/fit2000/final'][1]:.2f} dB (min view {gold[name + '/fit2000/per_view_psnr'].min():.2f})")
        # the loss went down by the same orders of magnitude as the reference's
        assert got["loss"][-1] <= 10.0 * gold[f"{name}/fit2000/loss"][-1] + 1e-6
    assert min_view["gaussian"] >= 35.0
    floor_db = min(finals["gaussian"], 35.0) - 2.0
    assert min(v for k, v in finals.items() if k != "gaussian") >= floor_db
    # the psi ablation: both runs qualify, as the reference's do on this start
    for tag, psi in (("calibrated", "default"), ("ablated", "1.0")):
        out = tmp_path / f"{tag}.txt"
        run(tool, "fit-scene", os.path.join(FIT, "scene.txt"), os.path.join(FIT, "cameras.txt"),
            os.path.join(FIT, "init_0.05.txt"), "half-cosine-sq", psi, 2000, out, timeout=1200)
        got = read_report(out)
        print(f"ablation {tag}: GPU {got['final'][1]:.2f} dB; reference {float(gold['ablation/' + tag + '/final_psnr']):.2f} dB")
        assert got["final"][1] >= 35.0


def test_acceptance_criterion_8_seeded_reruns_are_byte_identical(tool, tmp_path):
    """tests/acceptance.cpp:474-521 for the three subcommands on this path, in the deterministic
    mode (darbs_cuda_set_deterministic: order-independent fixed-point accumulation)."""
    outs = []
    for rep in ("a", "b"):
        d = tmp_path / rep
        d.mkdir()
        run(tool, "render", os.path.join(FIT, "scene.txt"), os.path.join(FIT, "cameras.txt"), "gaussian", "default", d)
        run(tool, "fit-scene", os.path.join(FIT, "scene.txt"), os.path.join(FIT, "cameras.txt"),
            os.path.join(FIT, "init_0.02.txt"), "gaussian", "default", 25, d / "fit_scene.txt", "deterministic")
        run(tool, "fit-image", os.path.join(FIT, "target2d.dsfl"), "gaussian", 40, 60, 5, d / "fit_image.txt",
            "deterministic")
        outs.append(d)
    names = sorted(os.listdir(outs[0]))
    assert names == sorted(os.listdir(outs[1])) and len(names) == 6
    for nm in names:
        assert (outs[0] / nm).read_bytes() == (outs[1] / nm).read_bytes(), nm


@pytest.mark.parametrize("name", ["gaussian", "half-cosine-sq", "raised-cosine"])
def test_fit_image_tracks_the_reference_trajectory(tool, gold, tmp_path, name):
    out = tmp_path / "fit2d.txt"
    run(tool, "fit-image", os.path.join(FIT, "target2d.dsfl"), name, 40, 60, 5, out)
    got = read_report(out)
    for key in ("loss", "l1", "dssim"):
        ref = gold[f"{name}/fit_image/{key}"]
        rel = np.abs(got[key] - ref) / np.abs(ref)
        assert rel.max() <= 1e-3, (name, key, int(rel.argmax()), rel.max())
    assert abs(got["final"][1] - gold[f"{name}/fit_image/final"][1]) <= 0.1
    splats = gold[f"{name}/fit_image/splats"]
    assert np.abs(got["rows"] - splats).max() <= 1e-3 * max(1.0, np.abs(splats).max())
