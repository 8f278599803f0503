#!/usr/bin/env python
"""Generates tests/golden/*.npz by running the REFERENCE'S OWN SOURCES.

The reference (arxiv/paper_2501_12369, proj/core) ships no golden images: every known answer in
its tests is closed-form or "reference vs its own brute-force oracle".  These
fixtures are therefore outputs of the reference itself: oracle/_ref/libdarbs_ref.so is
/root/reference/proj/core/src/{kernel,geometry,rasterizer,loss}.cpp compiled unmodified against
oracle/eigen_shim (oracle/Makefile `ref`).  /root/reference does not exist on the GPU box, so the
vectors are committed; this script is how they were made:

    make -C oracle ref && python tests/golden/make_golden.py

Every input is float32-representable (SURVEY.md §8c "parity input rule"), so the same numbers feed
the FP64 reference and the float32 C ABI.  Outputs are the reference's FP64 results.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import cpu  # noqa: E402

PRESETS = ["gaussian", "half-cosine-sq", "raised-cosine", "mod-sinc", "inv-multiquadratic"]
BG = (0.1, 0.2, 0.3)
# proj/data/demo_cameras.txt, first block (fx fy cx cy w h + 16 row-major world-to-camera)
DEMO_CAMERA = np.array([80, 80, 32, 32, 64, 64,
                        -0.3894183423, 0, 0.921060994, 4.278389336e-17,
                        -0.2646649291, 0.9578262852, -0.1118985373, -1.14366835e-16,
                        -0.8822164303, -0.2873478856, -0.3729951242, 3.132091953,
                        0, 0, 0, 1.0])


def f32r(a):
    return np.asarray(a, dtype=np.float32).astype(np.float64)


def raster_case(ref, name, n, w, h, seed):
    k = ref.preset(name)
    s = ref.random_scene(k, n, w, h, seed)
    g = ref.random_image_grad(w, h, 1000 + seed)
    offsets, plist, order = ref.bin(s, w, h)
    fr = ref.forward(k, s, w, h, BG, threads=1, keep=True)
    st, grads = ref.backward(fr["handle"], k, g, s, threads=1)
    ref.forward_free(fr["handle"])
    assert st == 0
    brute = ref.oracle_forward(k, s, w, h, BG)
    return dict(
        kernel=name, n=n, width=w, height=h, seed=seed, background=np.array(BG),
        mu2=s.mu2.astype(np.float32), cov2=s.cov2.astype(np.float32), conic=s.conic.astype(np.float32),
        radius=s.radius.astype(np.float32), depth=s.depth.astype(np.float32),
        opacity=s.opacity.astype(np.float32), rgb=s.rgb.astype(np.float32), grad_image=g.astype(np.float32),
        tile_offsets=offsets, point_list=plist, depth_order=order,
        image=fr["image"], t_final=fr["t_final"], processed=fr["processed"], contributors=fr["contributors"],
        skipped=fr["skipped"], brute_image=brute, splat_grads=grads)


def geometry_case(ref, name, n, seed):
    k = ref.preset(name)
    psi = ref.default_psi(name)
    rng = np.random.default_rng(seed)
    raw = np.zeros((n, 14))
    raw[:, 0:3] = rng.uniform(-0.9, 0.9, (n, 3))
    raw[:, 3:6] = np.log(rng.uniform(0.02, 0.08, (n, 3)))
    raw[:, 6:10] = rng.normal(size=(n, 4))
    raw[:, 10] = rng.normal(size=n)
    raw[:, 11:14] = rng.normal(size=(n, 3))
    raw[3, 0:3] = (3.5288, 1.1492, 1.4920)  # behind the demo camera: near-plane culled
    raw = f32r(raw)
    prims = f32r(ref.realize(raw))  # the float32 primitives the C ABI's project() consumes
    st, pr = ref.project(k, psi, prims, DEMO_CAMERA)
    assert st == 0
    gc = f32r(rng.normal(size=(n, 4)))
    gm = f32r(rng.normal(size=(n, 2)))
    d_mu, d_scale, d_rot = ref.backward_projection(psi, gc, gm, prims, DEMO_CAMERA)
    # the evaluate chain (fit3d.cpp:108-159) on the reference, fed float32-rounded splats
    prims_full = ref.realize(raw)
    st, pf = ref.project(k, psi, prims_full, DEMO_CAMERA)
    vis = np.flatnonzero(pf["valid"]).astype(np.int32)
    s = cpu.Scene(f32r(pf["mu2"][vis]), None, f32r(pf["conic"][vis]), pf["radius"][vis], f32r(pf["depth"][vis]),
                  f32r(prims_full[vis, 10]), f32r(prims_full[vis, 11:14]))
    w, h = 64, 64
    gimg = ref.random_image_grad(w, h, 77)
    fr = ref.forward(k, s, w, h, (0, 0, 0), threads=1, keep=True)
    st, sg = ref.backward(fr["handle"], k, gimg, s, threads=1)
    ref.forward_free(fr["handle"])
    pg = ref.param_grads(psi, vis, sg, s.conic, s.opacity, s.rgb, prims_full, DEMO_CAMERA)
    return dict(kernel=name, psi=psi, camera=DEMO_CAMERA, raw=raw.astype(np.float32),
                prims=prims.astype(np.float32), valid=pr["valid"], mu2=pr["mu2"], cov2=pr["cov2"],
                conic=pr["conic"], radius=pr["radius"], depth=pr["depth"],
                grad_cov2=gc.astype(np.float32), grad_mu2=gm.astype(np.float32), d_mu=d_mu, d_scale=d_scale,
                d_rot=d_rot, view_grad_image=gimg.astype(np.float32), view_image=fr["image"],
                view_param_grads=pg, view_processed=fr["processed"], view_contributors=fr["contributors"])


def eval_case(ref):
    out = {}
    for name in PRESETS:
        k = ref.preset(name)
        dm2 = f32r(np.concatenate([np.linspace(0.0, k.cutoff * 1.5, 257), [k.cutoff, 1e-20, 0.3, 1.0, 2.5, 8.9]]))
        st, w, dw = ref.eval(k, dm2)
        assert st == 0
        out[name + "/dm2"] = dm2.astype(np.float32)
        out[name + "/weight"] = w
        out[name + "/dweight"] = dw
        out[name + "/spec"] = np.array([k.family, k.beta, k.xi, k.lobes, k.cutoff, k.unbounded], dtype=np.float64)
        out[name + "/psi"] = np.array(ref.default_psi(name))
    return out


def adam_case(ref):
    rng = np.random.default_rng(3)
    dim = 14 * 64
    p = f32r(rng.normal(size=dim))
    g = f32r(rng.normal(size=dim))
    lrs = f32r(rng.uniform(1e-4, 1e-2, size=dim))
    m, v = np.zeros(dim), np.zeros(dim)
    out = dict(params0=p.astype(np.float32), grads=g.astype(np.float32), lrs=lrs.astype(np.float32))
    for t in (1, 2, 3):
        st, p, m, v = ref.adam_step(p, g, m, v, lrs, t)
        assert st == 0
        out[f"params{t}"], out[f"m{t}"], out[f"v{t}"] = p, m, v
    return out


def smooth_image(w, h, seed):
    """A renderer-like image: a few soft blobs on a gradient, float32-representable, in [0, 1]."""
    rng = np.random.default_rng(seed)
    yy, xx = np.mgrid[0:h, 0:w]
    img = np.zeros((h, w, 3))
    for _ in range(6):
        cx, cy, s = rng.uniform(0, w), rng.uniform(0, h), rng.uniform(2.0, 0.4 * max(w, h))
        img += np.exp(-((xx - cx) ** 2 + (yy - cy) ** 2) / (2 * s * s))[..., None] * rng.uniform(0, 0.6, 3)
    img += 0.2 * (xx / max(w - 1, 1))[..., None]
    return f32r(np.clip(img, 0.0, 1.0))


def loss_case(ref):
    """loss_total (loss.cpp:173-230) on the test fixture's random images (tests/test_loss.cpp:13-19)
    and on a smooth pair, at sizes that exercise single and repeated mirror reflection."""
    out = {}
    for tag, (w, h) in {"a": (10, 9), "b": (37, 21), "c": (3, 4), "d": (70, 45)}.items():
        x = ref.random_image(w, h, 3)
        y = ref.random_image(w, h, 4)
        if tag == "d":
            x = smooth_image(w, h, 5)
            y = f32r(np.clip(x + np.random.default_rng(6).normal(scale=0.02, size=x.shape), 0, 1))
        out[tag + "/rendered"], out[tag + "/target"] = x.astype(np.float32), y.astype(np.float32)
        for lam in (0.0, 0.2, 1.0):
            st, vals, grad = ref.loss_total(x, y, lam)
            assert st == 0
            out[f"{tag}/{lam}/values"] = np.array(vals)
            out[f"{tag}/{lam}/grad"] = grad
    return out


def io_fixtures(ref):
    """Files written by the reference's own writers (src/scene_io.cpp, src/image.cpp): the C++ mirror's
    readers and writers are byte-compared with them (tests/test_host_io.py)."""
    out = os.path.join(HERE, "io")
    os.makedirs(out, exist_ok=True)
    rng = np.random.default_rng(11)
    n = 12
    prims = np.zeros((n, 14))
    prims[:, 0:3] = rng.uniform(-1, 1, (n, 3))
    prims[:, 3:6] = rng.uniform(0.01, 0.3, (n, 3))
    prims[:, 6:10] = rng.normal(size=(n, 4))
    prims[:, 10] = rng.uniform(0, 1, n)
    prims[:, 11:14] = rng.uniform(0, 1, (n, 3))
    prims[0, 10], prims[1, 10] = 0.0, 1.0       # the closed ends of the opacity range
    prims[2, 0:3] = (1e-300, -2.5e17, 1.0 / 3)  # round trips need all 17 digits
    assert ref.write_scene(os.path.join(out, "scene.txt"), prims) == 0
    cams = np.stack([DEMO_CAMERA, DEMO_CAMERA])
    cams[1, 0:6] = (812.5, 799.25, 959.5, 539.5, 1920, 1080)
    cams[1, 6:22] += rng.normal(scale=1e-3, size=16)
    assert ref.write_cameras(os.path.join(out, "cameras.txt"), cams) == 0
    img = rng.uniform(-0.1, 1.1, (7, 9, 3))     # values outside [0, 1] exercise the PPM clamp
    img[0, 0] = (0.5 / 255.0, 1.5 / 255.0, 254.5 / 255.0)  # rounds half up
    assert ref.write_image(os.path.join(out, "image.dsfl"), img, ppm=False) == 0
    assert ref.write_image(os.path.join(out, "image.ppm"), img, ppm=True) == 0
    # what the PPM of the float dump must be: the dump stores float32, the clamp and rounding see those
    assert ref.write_image(os.path.join(out, "image_from_dsfl.ppm"), img.astype(np.float32).astype(np.float64),
                           ppm=True) == 0
    np.save(os.path.join(out, "scene_values.npy"), prims)


REF_DATA = "/root/reference/proj/data"
FIT_KERNELS = ["gaussian", "half-cosine-sq", "raised-cosine", "mod-sinc", "inv-multiquadratic"]


def perturbed(truth, amount, seed):
    """A seeded perturbation of the truth in the shape of tests/acceptance.cpp:391-405 (numpy's
    generator, not std::normal_distribution: the start is stored, so only its shape matters)."""
    rng = np.random.default_rng(seed)
    p = truth.copy()
    n = p.shape[0]
    p[:, 0:3] += amount * rng.normal(size=(n, 3))
    p[:, 3:6] *= np.exp(0.5 * amount * rng.normal(size=(n, 3)))
    p[:, 6:10] += 0.5 * amount * rng.normal(size=(n, 4))
    p[:, 10] = np.clip(p[:, 10] + 0.5 * amount * rng.normal(size=n), 0.02, 0.98)
    p[:, 11:14] = np.clip(p[:, 11:14] + 0.5 * amount * rng.normal(size=(n, 3)), 0.02, 0.98)
    return p


def fit_fixtures(ref):
    """The reference's own callers of the hot path — render_scene, fit_scene (src/fit3d.cpp) and
    fit_image (src/fit2d.cpp) — on its own data files proj/data/demo_scene.txt + demo_cameras.txt.
    Inputs are written by the reference's writers into tests/golden/fit/ (the C++ mirror reads
    them); results go to tests/golden/fit.npz.  tests/test_gpu_fit_drivers.py runs the mirror's
    fit_scene / fit_image / render_scene (host/fit_tool.cpp) on the same files on the GPU."""
    out = os.path.join(HERE, "fit")
    os.makedirs(out, exist_ok=True)
    n, truth = ref.read_scene(os.path.join(REF_DATA, "demo_scene.txt"))
    nc, cams = ref.read_cameras(os.path.join(REF_DATA, "demo_cameras.txt"))
    assert n == 20 and nc == 4
    assert ref.write_scene(os.path.join(out, "scene.txt"), truth) == 0
    assert ref.write_cameras(os.path.join(out, "cameras.txt"), cams) == 0
    res = {"truth": truth, "cameras": cams}
    inits = {}
    for amount in (0.02, 0.05):
        inits[amount] = perturbed(truth, amount, 1)
        assert ref.write_scene(os.path.join(out, f"init_{amount}.txt"), inits[amount]) == 0
        res[f"init_{amount}"] = inits[amount]

    for name in FIT_KERNELS:
        k, psi = ref.preset(name), ref.default_psi(name)
        # render (tools/main.cpp:336-351): every view of the demo scene
        views = [ref.render_scene(k, psi, truth, cam)[1] for cam in cams]
        res[f"{name}/render"] = np.stack(views)
        # targets as the float32 dumps both sides read (image.cpp:61-85)
        tdir = os.path.join(out, f"targets_{name}")
        os.makedirs(tdir, exist_ok=True)
        targets = [f32r(v) for v in views]
        for v, t in enumerate(targets):
            assert ref.write_image(os.path.join(tdir, f"view_{v}.dsfl"), t, ppm=False) == 0
        # 50-iteration trajectory from the stored start, on the stored targets
        st, r = ref.fit_scene(k, psi, inits[0.02], cams, targets, ref.fit_config(iters=50, seed=1))
        assert st == 0
        for key in ("loss", "l1", "dssim", "psnr", "per_view_psnr", "primitives"):
            res[f"{name}/fit50/{key}"] = r[key]
        res[f"{name}/fit50/final"] = np.array([r["final_mse"], r["final_psnr"], r["final_ssim"]])
        # acceptance criterion 7 (tests/acceptance.cpp:419-470): 2000 iterations, self-rendered targets
        st, r = ref.fit_scene(k, psi, inits[0.02], cams, views, ref.fit_config(iters=2000, seed=1))
        assert st == 0
        res[f"{name}/fit2000/final"] = np.array([r["final_mse"], r["final_psnr"], r["final_ssim"]])
        res[f"{name}/fit2000/per_view_psnr"] = r["per_view_psnr"]
        res[f"{name}/fit2000/loss"] = r["loss"]
        print(f"  fit_scene {name}: 50 it {res[name + '/fit50/final'][1]:.2f} dB, 2000 it {r['final_psnr']:.2f} dB "
              f"(min view {r['per_view_psnr'].min():.2f})", flush=True)
    # the psi ablation of criterion 7: half-cosine-sq, perturbation 0.05, fitted with psi and with 1.0
    k, psi = ref.preset("half-cosine-sq"), ref.default_psi("half-cosine-sq")
    views = [ref.render_scene(k, psi, truth, cam)[1] for cam in cams]
    for tag, psi_fit in (("calibrated", psi), ("ablated", 1.0)):
        st, r = ref.fit_scene(k, psi_fit, inits[0.05], cams, views, ref.fit_config(iters=2000, seed=1))
        assert st == 0
        res[f"ablation/{tag}/final_psnr"] = np.array(r["final_psnr"])
        print(f"  ablation {tag}: {r['final_psnr']:.2f} dB", flush=True)
    # fit_image (fit2d.cpp:45-188; the determinism criterion runs it with n = 40, 60 iterations, seed 5):
    # the target is view 0 of the Gaussian render
    target = f32r(res["gaussian/render"][0])
    assert ref.write_image(os.path.join(out, "target2d.dsfl"), target, ppm=False) == 0
    for name in ("gaussian", "half-cosine-sq", "raised-cosine"):
        st, r = ref.fit_image(ref.preset(name), target, 40, ref.fit_config(iters=60, seed=5))
        assert st == 0
        for key in ("loss", "l1", "dssim", "psnr", "splats", "rendered"):
            res[f"{name}/fit_image/{key}"] = r[key]
        res[f"{name}/fit_image/final"] = np.array([r["final_mse"], r["final_psnr"], r["final_ssim"]])
        print(f"  fit_image {name}: {r['final_psnr']:.2f} dB", flush=True)
    np.savez_compressed(os.path.join(HERE, "fit.npz"), **res)


def main():
    if len(sys.argv) > 1 and sys.argv[1] == "fit":  # only the drivers' fixtures
        fit_fixtures(cpu.load("reference"))
        return
    if not cpu.available("reference"):
        raise SystemExit("oracle/_ref/libdarbs_ref.so missing: run `make -C oracle ref` where /root/reference exists")
    ref = cpu.load("reference")
    assert ref.kind == "reference"
    for name in PRESETS:
        for seed, (n, w, h) in enumerate([(300, 48, 40), (150, 33, 17)]):
            np.savez_compressed(os.path.join(HERE, f"raster_{name}_{seed}.npz"), **raster_case(ref, name, n, w, h, seed))
    for name in ["gaussian", "half-cosine-sq", "raised-cosine", "inv-multiquadratic"]:
        np.savez_compressed(os.path.join(HERE, f"geometry_{name}.npz"), **geometry_case(ref, name, 120, 9))
    np.savez_compressed(os.path.join(HERE, "eval.npz"), **eval_case(ref))
    np.savez_compressed(os.path.join(HERE, "adam.npz"), **adam_case(ref))
    np.savez_compressed(os.path.join(HERE, "loss.npz"), **loss_case(ref))
    io_fixtures(ref)
    fit_fixtures(ref)
    total = sum(os.path.getsize(os.path.join(HERE, f)) for f in os.listdir(HERE) if f.endswith(".npz"))
    print(f"wrote golden fixtures, {total / 1024:.0f} KiB")


if __name__ == "__main__":
    main()
