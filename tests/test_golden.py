"""Golden vectors produced by the reference's own sources (tests/golden/make_golden.py).

CPU half (``-m "not gpu"``): the plain-C restatement reproduces every committed vector — this is
what pins the oracle on the GPU box, where /root/reference (and possibly oracle/_ref) is absent.
GPU half (``-m gpu``): the CUDA path through the C ABI reproduces the same vectors directly,
without any oracle in the loop.  Tolerances as in tests/test_gpu_rasterizer.py.
"""
import glob
import os

import numpy as np
import pytest

from conftest import f32, rel_err
from oracle.cpu import Scene

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
RASTER = sorted(glob.glob(os.path.join(GOLD, "raster_*.npz")))
GEOM = sorted(glob.glob(os.path.join(GOLD, "geometry_*.npz")))
IMG_TOL, GRAD_TOL = 2e-5, 1e-3


def ident(path):
    return os.path.basename(path)[:-4]


def test_fixtures_are_present():
    assert len(RASTER) == 10 and len(GEOM) == 4
    assert os.path.exists(os.path.join(GOLD, "eval.npz")) and os.path.exists(os.path.join(GOLD, "adam.npz"))


def gold_scene(z):
    return Scene(z["mu2"], z["cov2"], z["conic"], z["radius"], z["depth"], z["opacity"], z["rgb"])


# ----------------------------------------------------------------------------- CPU: the port
@pytest.mark.parametrize("path", RASTER, ids=ident)
def test_port_reproduces_raster_golden(port, path):
    z = np.load(path)
    k = port.preset(str(z["kernel"]))
    w, h, n, seed = int(z["width"]), int(z["height"]), int(z["n"]), int(z["seed"])
    s = port.random_scene(k, n, w, h, seed)  # the fixture generator itself is part of the restatement
    for f in ("mu2", "cov2", "conic", "radius", "depth", "opacity", "rgb"):
        assert np.array_equal(getattr(s, f), z[f].astype(np.float64)), f
    g = port.random_image_grad(w, h, 1000 + seed)
    assert np.array_equal(g, z["grad_image"].astype(np.float64))
    offsets, plist, order = port.bin(s, w, h)
    assert np.array_equal(offsets, z["tile_offsets"])
    assert np.array_equal(plist, z["point_list"])
    assert np.array_equal(order, z["depth_order"])
    fr = port.forward(k, s, w, h, tuple(z["background"]), keep=True)
    assert np.array_equal(fr["processed"], z["processed"])
    assert np.array_equal(fr["contributors"], z["contributors"])
    assert fr["skipped"] == int(z["skipped"])
    assert np.abs(fr["image"] - z["image"]).max() <= 1e-12
    assert np.abs(fr["t_final"] - z["t_final"]).max() <= 1e-12
    assert np.abs(port.oracle_forward(k, s, w, h, tuple(z["background"])) - z["brute_image"]).max() <= 1e-12
    st, grads = port.backward(fr["handle"], k, g, s)
    port.forward_free(fr["handle"])
    assert st == 0
    assert np.abs(grads - z["splat_grads"]).max() <= 1e-11 * max(1.0, np.abs(z["splat_grads"]).max())


@pytest.mark.parametrize("path", GEOM, ids=ident)
def test_port_reproduces_geometry_golden(port, path):
    z = np.load(path)
    k = port.preset(str(z["kernel"]))
    psi, cam = float(z["psi"]), z["camera"]
    prims = z["prims"].astype(np.float64)
    st, pr = port.project(k, psi, prims, cam)
    assert st == 0
    assert np.array_equal(pr["valid"], z["valid"]) and pr["valid"].sum() < prims.shape[0]
    assert np.array_equal(pr["radius"], z["radius"])
    for f in ("mu2", "cov2", "conic", "depth"):
        assert np.abs(pr[f] - z[f]).max() <= 1e-11 * max(1.0, np.abs(z[f]).max()), f
    out = port.backward_projection(psi, z["grad_cov2"].astype(np.float64), z["grad_mu2"].astype(np.float64), prims, cam)
    for a, f in zip(out, ("d_mu", "d_scale", "d_rot")):
        assert np.abs(a - z[f]).max() <= 1e-10 * max(1.0, np.abs(z[f]).max()), f
    # the per-view evaluate chain, fit3d.cpp:108-159
    raw = z["raw"].astype(np.float64)
    full = port.realize(raw)
    st, pf = port.project(k, psi, full, cam)
    vis = np.flatnonzero(pf["valid"]).astype(np.int32)
    r32 = lambda a: a.astype(np.float32).astype(np.float64)  # noqa: E731
    s = Scene(r32(pf["mu2"][vis]), None, r32(pf["conic"][vis]), pf["radius"][vis], r32(pf["depth"][vis]),
              r32(full[vis, 10]), r32(full[vis, 11:14]))
    fr = port.forward(k, s, 64, 64, (0, 0, 0), keep=True)
    st, sg = port.backward(fr["handle"], k, z["view_grad_image"].astype(np.float64), s)
    port.forward_free(fr["handle"])
    pg = port.param_grads(psi, vis, sg, s.conic, s.opacity, s.rgb, full, cam)
    assert np.array_equal(fr["processed"], z["view_processed"])
    assert np.abs(fr["image"] - z["view_image"]).max() <= 1e-12
    assert np.abs(pg - z["view_param_grads"]).max() <= 1e-9 * max(1.0, np.abs(z["view_param_grads"]).max())


def test_port_reproduces_eval_and_adam_golden(port):
    z = np.load(os.path.join(GOLD, "eval.npz"))
    for name in ("gaussian", "half-cosine-sq", "raised-cosine", "mod-sinc", "inv-multiquadratic"):
        k = port.preset(name)
        spec = z[name + "/spec"]
        assert (k.family, k.beta, k.xi, k.lobes, k.cutoff, k.unbounded) == tuple(spec)
        assert port.default_psi(name) == float(z[name + "/psi"])
        st, w, dw = port.eval(k, z[name + "/dm2"].astype(np.float64))
        assert st == 0
        assert np.abs(w - z[name + "/weight"]).max() <= 1e-15
        assert np.abs(dw - z[name + "/dweight"]).max() <= 1e-14
    z = np.load(os.path.join(GOLD, "adam.npz"))
    p, m, v = z["params0"].astype(np.float64), np.zeros(z["params0"].size), np.zeros(z["params0"].size)
    for t in (1, 2, 3):
        st, p, m, v = port.adam_step(p, z["grads"].astype(np.float64), m, v, z["lrs"].astype(np.float64), t)
        assert np.abs(p - z[f"params{t}"]).max() <= 1e-15
        assert np.abs(m - z[f"m{t}"]).max() <= 1e-15 and np.abs(v - z[f"v{t}"]).max() <= 1e-15


LOSS_TAGS = ("a", "b", "c", "d")


def test_port_reproduces_loss_golden(port):
    z = np.load(os.path.join(GOLD, "loss.npz"))
    for tag in LOSS_TAGS:
        x, y = z[tag + "/rendered"].astype(np.float64), z[tag + "/target"].astype(np.float64)
        for lam in (0.0, 0.2, 1.0):
            st, vals, grad = port.loss_total(x, y, lam)
            assert st == 0
            assert np.abs(np.array(vals) - z[f"{tag}/{lam}/values"]).max() <= 1e-13
            assert np.abs(grad - z[f"{tag}/{lam}/grad"]).max() <= 1e-15


# ----------------------------------------------------------------------------- GPU: the C ABI
@pytest.mark.parametrize("name", ["gaussian", "half-cosine-sq", "raised-cosine", "mod-sinc", "inv-multiquadratic"])
def test_port_reproduces_the_first_iteration_of_the_reference_fit(port, name):
    """tests/golden/fit.npz holds the reference's own fit_scene runs on its demo scene (made by
    make_golden.py through oracle/_ref).  Its first recorded loss is fit3d.cpp:108-165 evaluated at the
    stored start: the port's project -> forward -> loss_total over the four demo cameras must give
    the same mean (this pins the fixture the GPU drivers are compared with, without a GPU), and the
    port's render of the truth must be the stored reference render."""
    z = np.load(os.path.join(GOLD, "fit.npz"))
    k, psi = port.preset(name), port.default_psi(name)
    cams, truth, init = z["cameras"], z["truth"], z["init_0.02"]
    sums = np.zeros(3)
    for v, cam in enumerate(cams):
        w, h = int(cam[4]), int(cam[5])

        def render(prims):
            st, pr = port.project(k, psi, prims, cam)
            assert st == 0
            vis = np.flatnonzero(pr["valid"])
            s = Scene(pr["mu2"][vis], None, pr["conic"][vis], pr["radius"][vis], pr["depth"][vis], prims[vis, 10],
                      prims[vis, 11:14])
            return port.forward(k, s, w, h, (0, 0, 0), threads=0)["image"]

        ref_render = z[f"{name}/render"][v]
        assert np.abs(render(truth) - ref_render).max() <= 1e-12
        target = ref_render.astype(np.float32).astype(np.float64)  # the float32 dumps both sides read
        st, vals, _ = port.loss_total(render(init), target, 0.2, want_grad=False)
        sums += vals
    mean = sums / len(cams)
    assert abs(mean[0] - z[f"{name}/fit50/loss"][0]) <= 1e-12
    assert abs(mean[1] - z[f"{name}/fit50/l1"][0]) <= 1e-12
    assert abs(mean[2] - z[f"{name}/fit50/dssim"][0]) <= 1e-12


@pytest.mark.gpu
@pytest.mark.parametrize("path", RASTER, ids=ident)
def test_gpu_reproduces_raster_golden(ctx, darbs, path):
    z = np.load(path)
    gk = darbs.kernel_preset(str(z["kernel"]))
    w, h, n = int(z["width"]), int(z["height"]), int(z["n"])
    b = ctx.bin(z["mu2"], z["conic"], z["radius"], z["depth"], w, h)
    offsets = z["tile_offsets"]
    assert b["num_entries"] == z["point_list"].size
    assert np.array_equal(b["point_list"], z["point_list"])
    assert np.array_equal(b["depth_order"], z["depth_order"])
    assert np.array_equal(b["tile_ranges"][:, 1] - b["tile_ranges"][:, 0], np.diff(offsets))
    out = ctx.forward(gk, z["mu2"], z["conic"], z["radius"], z["depth"], z["opacity"], z["rgb"], w, h,
                      tuple(z["background"]))
    assert np.array_equal(out["processed"], z["processed"])
    assert np.array_equal(out["contributors"], z["contributors"])
    assert out["skipped"] == int(z["skipped"])
    assert np.abs(out["image"] - z["image"]).max() <= IMG_TOL
    assert np.abs(out["image"] - z["brute_image"]).max() <= IMG_TOL
    assert np.abs(out["t_final"] - z["t_final"]).max() <= IMG_TOL
    grads = ctx.backward(gk, z["grad_image"], n)
    ref = z["splat_grads"]
    floor = np.maximum(1e-4, 1e-3 * np.abs(ref).max(axis=0, keepdims=True))
    assert rel_err(grads, ref, floor).max() <= GRAD_TOL


@pytest.mark.gpu
@pytest.mark.parametrize("path", GEOM, ids=ident)
def test_gpu_reproduces_geometry_golden(ctx, darbs, path):
    z = np.load(path)
    gk = darbs.kernel_preset(str(z["kernel"]))
    psi, cam = float(z["psi"]), z["camera"]
    g = ctx.project(gk, psi, z["prims"], cam)
    assert np.array_equal(g["valid"], z["valid"])
    v = z["valid"] == 1
    assert np.array_equal(g["radius"][v], z["radius"][v])
    for f in ("mu2", "cov2", "conic", "depth"):
        assert rel_err(g[f][v], z[f][v], 1e-3).max() <= 1e-6, f
    out = ctx.backward_projection(psi, z["grad_cov2"], z["grad_mu2"], z["prims"], cam)
    for a, f in zip(out, ("d_mu", "d_scale", "d_rot")):
        assert np.abs(a - z[f]).max() <= 1e-5 * np.abs(z[f]).max(), f
    n = z["raw"].shape[0]
    pg = np.zeros((n, 14), np.float32)
    img = np.zeros((64, 64, 3), np.float32)
    ctx.evaluate_view(gk, psi, z["raw"], cam, (0, 0, 0), grad_image=z["view_grad_image"], param_grads=pg,
                      image_out=img)
    ref = z["view_param_grads"]
    assert np.abs(img - z["view_image"]).max() <= 5e-5
    assert rel_err(pg, ref, 1e-4 * max(1.0, np.abs(ref).max())).max() <= 2e-3


@pytest.mark.gpu
def test_gpu_reproduces_eval_and_adam_golden(ctx, darbs):
    z = np.load(os.path.join(GOLD, "eval.npz"))
    for name in ("gaussian", "half-cosine-sq", "raised-cosine", "mod-sinc", "inv-multiquadratic"):
        gk = darbs.kernel_preset(name)
        assert (gk.family, gk.beta, gk.xi, gk.lobes, gk.cutoff, gk.unbounded) == tuple(z[name + "/spec"])
        assert darbs.default_psi(name) == float(z[name + "/psi"])
        w, dw = ctx.eval(gk, z[name + "/dm2"])
        assert np.abs(w - z[name + "/weight"]).max() <= 2e-6
        assert np.abs(dw - z[name + "/dweight"]).max() <= 1e-5 * max(1.0, np.abs(z[name + "/dweight"]).max())
    z = np.load(os.path.join(GOLD, "adam.npz"))
    p = z["params0"].copy()
    m, v = np.zeros(p.size, np.float32), np.zeros(p.size, np.float32)
    for t in (1, 2, 3):
        ctx.adam_step(p, f32(z["grads"]), m, v, f32(z["lrs"]), t)
        assert np.abs(p - z[f"params{t}"]).max() <= 1e-6


@pytest.mark.gpu
def test_gpu_reproduces_loss_golden(ctx):
    """loss_total through the C ABI against the reference's own outputs.  Tolerances: values 2e-6
    absolute (FP32 moments, FP64 sums); gradient max |g - g_ref| <= 1e-5 max |g_ref| and
    |g - g_ref| <= 1e-3 max(|g|, |g_ref|, floor) with floor = 1e-2 of the largest reference gradient."""
    z = np.load(os.path.join(GOLD, "loss.npz"))
    for tag in LOSS_TAGS:
        x, y = z[tag + "/rendered"], z[tag + "/target"]
        for lam in (0.0, 0.2, 1.0):
            vals, grad = ctx.loss_total(x, y, lam)
            ref_vals, ref_grad = z[f"{tag}/{lam}/values"], z[f"{tag}/{lam}/grad"]
            assert np.abs(np.array(vals[:3]) - ref_vals).max() <= 2e-6
            assert np.abs(grad - ref_grad).max() <= 1e-5 * np.abs(ref_grad).max()
            assert rel_err(grad, ref_grad, 1e-2 * np.abs(ref_grad).max()).max() <= 1e-3
