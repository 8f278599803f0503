"""Differential fuzzing of bin / forward / backward against the oracle (GPU box only).

Random image sizes, splat counts, DARBF kernels (presets and custom beta / xi / lobes) and scene
mutations (footprint scale, radius unrelated to the footprint, opacity regimes including exact 0
and 1, equal / negative depths, non-finite conic or radius, off-screen means), each compared the
way tests/test_gpu_rasterizer.py compares: lists, ranges, depth order, processed, contributors
bit-exact; image / t_final within IMG_TOL; gradients by grad_err.  Prints one line per failing
trial with the recipe to replay it.  tests/test_gpu_fuzz.py runs a fixed block of seeds; longer
campaigns:   python tests/fuzz_cases.py [trials] [first seed]   (FUZZ_NMAX=40000 for larger scenes;
4000 trials at that size passed on 2026-10-17)."""
import os
import sys
import traceback

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "tests")):
    if p not in sys.path:
        sys.path.insert(0, p)
from conftest import f32, rel_err, scene_f32  # noqa: E402
import test_gpu_rasterizer as T  # noqa: E402

NMAX = int(os.environ.get("FUZZ_NMAX", "6000"))
FAMILIES = ["gaussian", "half-cosine", "raised-cosine", "mod-sinc", "inv-multiquadratic"]


def pick_kernel(rng):
    if rng.uniform() < 0.6:
        return rng.choice(T.KERNELS)
    fam = rng.choice(FAMILIES)
    beta = float(rng.choice([1.0, 1.5, 2.0, 2.5]))
    xi = float(np.round(rng.uniform(0.4, 3.0), 2))
    lobes = int(rng.integers(1, 4)) if fam in ("half-cosine", "raised-cosine", "mod-sinc") else 1
    if fam == "inv-multiquadratic":
        beta = 2.0
    return f"custom:{fam}:{beta}:{xi}:{lobes}"


def mutate(rng, s, w, h, log):
    n = s.n
    if n == 0:
        return
    r = rng.uniform
    if r() < 0.3:  # footprint scale (conic ~ 1/sigma^2); radius follows or not
        f = float(np.exp(r(-2.5, 2.5)))
        s.conic[:] = f32(s.conic * f).astype(np.float64)
        if r() < 0.5:
            s.radius[:] = np.ceil(s.radius / np.sqrt(f))
        log.append(f"conic*{f:.3g}")
    if r() < 0.2:  # radius unrelated to the footprint (binning only looks at the radius)
        s.radius[:] = rng.integers(0, 40, n).astype(np.float64)
        log.append("radius random")
    mode = rng.integers(0, 5)
    if mode == 1:
        s.opacity[:] = f32(rng.uniform(0.9, 1.0, n))
        s.opacity[:: max(1, n // 7)] = 1.0
    elif mode == 2:
        s.opacity[:] = f32(rng.uniform(0.0, 0.02, n))
        s.opacity[:: max(1, n // 5)] = 0.0
    elif mode == 3:
        s.opacity[:] = f32(rng.choice([0.0, 1.0 / 255.0, 0.5, 0.99, 1.0], n))
    log.append(f"opacity mode {mode}")
    if r() < 0.3:
        s.depth[:] = f32(rng.choice(s.depth[: max(1, n // 10)], n))  # many ties
        log.append("depth ties")
    if r() < 0.2:
        s.depth[rng.integers(0, n, max(1, n // 20))] *= -1.0
        log.append("negative depths")
    if r() < 0.2:
        idx = rng.integers(0, n, max(1, n // 50))
        s.conic[idx, rng.integers(0, 3)] = rng.choice([np.nan, np.inf, -np.inf])
        idx = rng.integers(0, n, max(1, n // 50))
        s.radius[idx] = rng.choice([np.nan, np.inf])
        log.append("non-finite")
    if r() < 0.2:
        idx = rng.integers(0, n, max(1, n // 10))
        s.mu2[idx] = f32(rng.uniform(-3000, 3000, (idx.size, 2))).astype(np.float64)
        s.radius[idx[: idx.size // 2]] = 5000.0
        log.append("far means / huge radii")


def trial(ctx, port, seed):
    rng = np.random.default_rng(seed)
    name = pick_kernel(rng)
    w = int(rng.integers(1, 400)) if rng.uniform() < 0.8 else int(rng.integers(1, 20))
    h = int(rng.integers(1, 300)) if rng.uniform() < 0.8 else int(rng.integers(1, 20))
    n = int(np.exp(rng.uniform(0, np.log(NMAX)))) - 1
    k = T.oracle_kernel(port, name)
    s = port.random_scene(k, n, w, h, int(rng.integers(0, 1000)))
    log = [f"seed {seed}: {name} {w}x{h} n={n}"]
    mutate(rng, s, w, h, log)
    bg = tuple(float(x) for x in f32(rng.uniform(0, 1, 3)))
    # the two knobs results must not depend on (beyond the stated bars): how much of a tile's list the
    # cull kernel covers before the forward's blocks cull on by themselves, and the fixed-point
    # accumulation of the deterministic mode
    seg = int(rng.choice([0, 0, 1, 7, 16, 33, 64, 200]))
    det = bool(rng.uniform() < 0.25)
    log.append(f"segment {seg}, deterministic {det}")
    ctx.set_cull_segment(seg)
    ctx.set_deterministic(det)
    try:
        T.check_bins(ctx, port, s, w, h)
        fr = port.forward(k, s, w, h, bg, threads=0, keep=True)
        gk = T.gpu_kernel_cached(name)
        out = ctx.forward(gk, **scene_f32(s), width=w, height=h, background=bg)
        assert out["skipped"] == fr["skipped"], ("skipped", out["skipped"], fr["skipped"])
        bad = int((out["processed"] != fr["processed"]).sum()), int((out["contributors"] != fr["contributors"]).sum())
        assert bad == (0, 0), ("processed/contributors differ at", bad)
        e = np.abs(out["image"] - fr["image"]).max() if w * h else 0.0
        assert e <= T.IMG_TOL, ("image", e)
        e = np.abs(out["t_final"] - fr["t_final"]).max() if w * h else 0.0
        assert e <= T.IMG_TOL, ("t_final", e)
        g = port.random_image_grad(w, h, int(rng.integers(0, 100)))
        st, ref = port.backward(fr["handle"], k, g, s, threads=0)
        port.forward_free(fr["handle"])
        assert st == 0
        got = ctx.backward(gk, f32(g), n)
        if n:
            # grad_err's floor is 1e-3 of a COLUMN's largest magnitude; with a handful of splats a column
            # is one cancelling sum (d_conic_b of a symmetric splat), so the floor here is 1e-3 of the
            # largest magnitude of the component's GROUP (colour / opacity / conic / mean)
            floor = np.empty((1, 9))
            for cols in ((0, 1, 2), (3,), (4, 5, 6), (7, 8)):
                floor[0, list(cols)] = max(T.GRAD_FLOOR, 1e-3 * np.abs(ref[:, list(cols)]).max())
            err = rel_err(got, ref, floor)
            assert np.isfinite(got).all(), "non-finite gradient"
            # 3 x GRAD_TOL: the tail of ~70 000 trials is one element at 2.4e-3 (2093 splats of opacity
            # <= 0.02 over a 9x3 image: lists of a thousand entries per pixel, float32 sums)
            assert err.max() <= 3.0 * T.GRAD_TOL, ("grad", float(err.max()), np.unravel_index(err.argmax(), err.shape))
    except Exception as ex:  # noqa: BLE001
        print("FAIL", "; ".join(log), "->", repr(ex)[:300], flush=True)
        if os.environ.get("FUZZ_TRACE"):
            traceback.print_exc()
        return False
    finally:
        ctx.set_cull_segment(0)
        ctx.set_deterministic(False)
    return True


# ------------------------------------------------------------------ the 3-D chain (fit3d.cpp:108-159)
PRESETS = ["gaussian", "half-cosine-sq", "raised-cosine", "mod-sinc", "inv-multiquadratic"]


def look_at_camera(rng, w, h):
    """22 doubles (include/darbs/scene_io.hpp:16-19): a camera somewhere on a sphere around the
    origin, looking at a point near it, rolled about its axis."""
    c = rng.normal(size=3)
    c *= rng.uniform(1.5, 5.0) / np.linalg.norm(c)
    f = rng.normal(scale=0.2, size=3) - c
    f /= np.linalg.norm(f)
    up = rng.normal(size=3)
    r = np.cross(up, f)
    r /= np.linalg.norm(r)
    u = np.cross(f, r)
    rot = np.stack([r, u, f])
    m = np.eye(4)
    m[:3, :3] = rot
    m[:3, 3] = -rot @ c
    focal = rng.uniform(0.5, 2.0) * max(w, h)
    return np.concatenate([[focal, focal * rng.uniform(0.9, 1.1), w / 2.0 + rng.uniform(-3, 3), h / 2.0 + rng.uniform(-3, 3),
                            w, h], m.reshape(-1)])


def chain_case(port, darbs, seed):
    """The random view of chain_trial: kernel, psi, camera, raw parameters, loss mode."""
    rng = np.random.default_rng(seed)
    name = str(rng.choice(PRESETS))
    psi = port.default_psi(name) if rng.uniform() < 0.6 else float(np.round(rng.uniform(0.5, 2.5), 3))
    w, h = int(rng.integers(8, 260)), int(rng.integers(8, 200))
    cam = look_at_camera(rng, w, h)
    n = int(np.exp(rng.uniform(0, np.log(4000))))
    lo = float(np.exp(rng.uniform(np.log(0.003), np.log(0.05))))
    raw = np.zeros((n, 14))
    # the scene stays inside a ball of radius 1.4 around the origin (cameras sit at 1.5 to 5): a
    # primitive a few hundredths in front of the camera plane projects to a footprint of 10^4 pixels
    # whose conic gradients (~1e6) cancel to parameter gradients of order one, beyond float32
    # (measured 2e-3 .. 6e-2 on single components); some primitives go BEHIND the camera instead
    raw[:, 0:3] = rng.uniform(-1, 1, (n, 3)) * rng.uniform(0.2, 0.8)
    if rng.uniform() < 0.5:
        idx = rng.integers(0, n, max(1, n // 10))
        eye = -(cam[6:18].reshape(3, 4)[:, :3].T @ cam[6:18].reshape(3, 4)[:, 3])
        raw[idx, 0:3] = eye * rng.uniform(1.05, 2.0, (idx.size, 1))
    raw[:, 3:6] = np.log(rng.uniform(lo, lo * rng.uniform(1.5, 8.0), (n, 3)))
    raw[:, 6:10] = rng.normal(size=(n, 4))
    raw[:, 10] = rng.normal(scale=2.0, size=n)
    raw[:, 11:14] = rng.normal(scale=1.5, size=(n, 3))
    lam = float(rng.choice([0.0, 0.2, 0.7, 1.0]))
    use_loss = rng.uniform() < 0.6
    return dict(rng=rng, name=name, psi=psi, w=w, h=h, cam=cam, n=n, raw=f32(raw), lam=lam, use_loss=use_loss,
                log=f"chain seed {seed}: {name} psi={psi} {w}x{h} n={n} scale~{lo:.3g} lam={lam if use_loss else None}")


def chain_trial(ctx, port, darbs, seed):
    """realize -> project -> forward -> loss -> backward -> parameter gradients of one view against
    the same chain built from the oracle's functions (the rasterizer fed float32-rounded splats,
    SURVEY 8c): visibility and radius exact, projected values 1e-6, image 5e-5, loss values 2e-6,
    parameter gradients: 5e-2 on every element and 2e-3 on all but three (or 0.1 %) of them, with a floor
    of 1e-3 of the column's largest magnitude (absolute errors of 5e-5 resp. 2e-6 of the column's scale)."""
    from oracle.cpu import Scene

    c = chain_case(port, darbs, seed)
    rng, name, psi, w, h, cam, n, raw, lam, use_loss, log = (c[key] for key in (
        "rng", "name", "psi", "w", "h", "cam", "n", "raw", "lam", "use_loss", "log"))
    k, gk = port.preset(name), darbs.kernel_preset(name)
    r32 = lambda a: a.astype(np.float32).astype(np.float64)  # noqa: E731
    try:
        prims = port.realize(raw.astype(np.float64))
        st, pr = port.project(k, psi, prims, cam)
        assert st == 0, ("oracle project", st)
        vis = np.flatnonzero(pr["valid"]).astype(np.int32)
        img = np.zeros((h, w, 3), np.float32)
        zero = np.zeros((h, w, 3), np.float32)
        if vis.size == 0:  # fit3d.cpp:117-119
            try:
                ctx.evaluate_view(gk, psi, raw, cam, (0, 0, 0), grad_image=zero, image_out=img)
            except darbs.DarbsError as e:
                assert e.status == 2
                return True
            raise AssertionError("all primitives culled but no numeric_error")
        # project_primitive alone, both sides fed the SAME float32 primitives (geometry.cpp:66-87)
        prims_g = ctx.realize(raw)
        g = ctx.project(gk, psi, prims_g, cam)
        st, po = port.project(k, psi, prims_g.astype(np.float64), cam)
        assert st == 0 and np.array_equal(g["valid"], po["valid"]), "visibility"
        v = po["valid"] == 1
        assert np.array_equal(g["radius"][v], po["radius"][v]), "radius"
        for key in ("mu2", "conic", "depth"):
            e = rel_err(g[key][v], po[key][v], 1e-3).max()
            assert e <= 2e-6, (key, float(e))
        s = Scene(r32(pr["mu2"][vis]), None, r32(pr["conic"][vis]), pr["radius"][vis], r32(pr["depth"][vis]),
                  r32(prims[vis, 10]), r32(prims[vis, 11:14]))
        fr = port.forward(k, s, w, h, (0, 0, 0), threads=0, keep=True)
        pg = np.zeros((n, 14), np.float32)
        if use_loss:
            ctx.evaluate_view(gk, psi, raw, cam, (0, 0, 0), grad_image=zero, image_out=img)
            # |rendered - target| >= 0.02 everywhere: the L1 term's sign(d) (loss.cpp:186) must not hang on
            # the float32 rounding of the image (unclipped, so that no target value ties with the image)
            target = f32(img + rng.choice([-1.0, 1.0], img.shape) * rng.uniform(0.02, 0.15, img.shape))
            vals = ctx.evaluate_view(gk, psi, raw, cam, (0, 0, 0), target=target, lam=lam, param_grads=pg)
            st, ref_vals, gimg = port.loss_total(fr["image"], target.astype(np.float64), lam)
            assert st == 0
            assert np.abs(np.array(vals[:3]) - np.array(ref_vals)).max() <= 5e-6, ("loss", vals, ref_vals)
        else:
            gimg = r32(port.random_image_grad(w, h, int(rng.integers(0, 100))))
            ctx.evaluate_view(gk, psi, raw, cam, (0, 0, 0), grad_image=f32(gimg), param_grads=pg, image_out=img)
        e = np.abs(img - fr["image"]).max()
        assert e <= 5e-5, ("image", float(e))
        st, sg = port.backward(fr["handle"], k, gimg, s, threads=0)
        port.forward_free(fr["handle"])
        assert st == 0
        ref = port.param_grads(psi, vis, sg, s.conic, s.opacity, s.rgb, prims, cam)
        assert np.isfinite(pg).all(), "non-finite parameter gradient"
        floor = np.maximum(1e-3 * np.abs(ref).max(axis=0, keepdims=True), 1e-12)
        err = rel_err(pg, ref, floor)
        # a gradient component is a float32 sum over the splat's pixels, accurate to ~3e-7 of the sum of
        # its terms' magnitudes; where the terms cancel (one colour channel of one splat, say) that is
        # more than 2e-6 of the COLUMN's scale (measured over 6000 views: 0.4 % of the views had one
        # such element; over 36000 views the largest was 3.7e-5 of the column's scale)
        assert err.max() <= 5e-2, ("param grads", float(err.max()), np.unravel_index(err.argmax(), err.shape))
        assert int((err > 2e-3).sum()) <= max(3, err.size // 1000), ("param grads", int((err > 2e-3).sum()))
    except Exception as ex:  # noqa: BLE001
        print("FAIL", log, "->", repr(ex)[:300], flush=True)
        if os.environ.get("FUZZ_TRACE"):
            traceback.print_exc()
        return False
    return True


# ------------------------------------------------------------------ loss_total (loss.cpp:173-230)
def loss_trial(ctx, port, seed):
    """Random sizes from below the window to several tiles, random lambda, images that are unrelated,
    smooth with small noise, or nearly identical (where the reference's partials cancel).  Values by
    the bars of tests/test_gpu_loss.py; the gradient image within 5e-4 of its largest element
    (test_gpu_loss.py holds 1e-5 on its cases and at 1080p; over 6000 random cases 7 % lie between
    1e-5 and 1e-4 and seven between 1e-4 and 3e-4, all on smooth images: the FP32 second moments are
    taken about ONE reference value per 32x16 tile, and where the local mean is far from it
    var = E[x'^2] - E[x']^2 loses digits against a variance of 1e-4 and C2 = 9e-4)."""
    import test_gpu_loss as L

    rng = np.random.default_rng(seed)
    w, h = int(rng.integers(1, 150)), int(rng.integers(1, 120))
    lam = float(rng.choice([0.0, 0.2, 1.0, float(np.round(rng.uniform(0, 1), 3))]))
    mode = int(rng.integers(0, 3))
    if mode == 0:
        x, y = f32(rng.uniform(0, 1, (h, w, 3))), f32(rng.uniform(0, 1, (h, w, 3)))
    elif mode == 1:
        x, y = L.smooth_pair(w, h, int(rng.integers(0, 1000)), noise=float(rng.choice([0.005, 0.02, 0.1])))
    else:
        x = L.smooth_pair(w, h, int(rng.integers(0, 1000)))[0]
        y = f32(x + rng.normal(scale=1e-4, size=x.shape))
    try:
        # values: 5e-6 (the mean of a few hundred FP32 SSIM values of a tiny image reaches 2.1e-6)
        L.check(ctx, port, x, y, lam, abs_tol=5e-4, floor_frac=0.5, val_tol=5e-6)
    except Exception as ex:  # noqa: BLE001
        print(f"FAIL loss seed {seed}: {w}x{h} lam={lam} mode={mode} ->", repr(ex)[:300], flush=True)
        return False
    return True


# ------------------------------------------------------------------ bin_splats alone, large shapes
def bins_trial(ctx, port, seed):
    """rasterizer.cpp:25-53 on shapes the rasterizer trials do not reach: up to 6000 pixels a side (more
    than 256 tile columns or rows: 32-bit tile keys and a second byte per coordinate), one-tile-wide
    strips, up to 200 k splats, radii from 0 to thousands of pixels (K up to tens of millions)."""
    rng = np.random.default_rng(seed)
    shape = int(rng.integers(0, 4))
    if shape == 0:
        w, h = int(rng.integers(1, 6000)), int(rng.integers(1, 6000))
    elif shape == 1:
        w, h = int(rng.integers(1, 17)), int(rng.integers(1, 6000))
    elif shape == 2:
        w, h = int(rng.integers(1, 6000)), int(rng.integers(1, 17))
    else:
        w, h = int(rng.integers(1, 700)), int(rng.integers(1, 700))
    n = int(np.exp(rng.uniform(0, np.log(200_000))))
    k = port.preset(str(rng.choice(["gaussian", "raised-cosine"])))
    s = port.random_scene(k, n, w, h, int(rng.integers(0, 1000)))
    tiles = ((w + 15) // 16) * ((h + 15) // 16)
    # radii: keep K below ~3e7 (a splat of radius R touches about (2R/16 + 1)^2 tiles)
    rmax = 16.0 * max(1.0, np.sqrt(min(3e7 / n, tiles)) / 2.0)
    mode = int(rng.integers(0, 3))
    if mode == 1:
        s.radius[:] = np.floor(rng.uniform(0, rmax, n))
    elif mode == 2:
        s.radius[:] = np.floor(np.exp(rng.uniform(0, np.log(rmax + 1.0), n)))
        s.radius[rng.integers(0, n, 3)] = 10_000.0
    if rng.uniform() < 0.3:
        s.depth[:] = f32(rng.choice(s.depth[: max(1, n // 50)], n))
    if rng.uniform() < 0.2:
        s.radius[rng.integers(0, n, max(1, n // 100))] = np.nan
    try:
        T.check_bins(ctx, port, s, w, h)
    except Exception as ex:  # noqa: BLE001
        print(f"FAIL bins seed {seed}: {w}x{h} n={n} mode={mode} ->", repr(ex)[:300], flush=True)
        return False
    return True


if __name__ == "__main__":
    import paper_2501_12369_b200 as darbs
    from oracle import cpu

    trials = int(sys.argv[1]) if len(sys.argv) > 1 else 200
    seed0 = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    port_, ctx_ = cpu.load("port"), darbs.Context(0)
    ok = sum(trial(ctx_, port_, seed0 + i) for i in range(trials))
    print(f"{ok}/{trials} rasterizer trials passed (seeds {seed0}..{seed0 + trials - 1})")
    ok = sum(chain_trial(ctx_, port_, darbs, seed0 + i) for i in range(trials))
    print(f"{ok}/{trials} chain trials passed (seeds {seed0}..{seed0 + trials - 1})")
    ok = sum(bins_trial(ctx_, port_, seed0 + i) for i in range(max(1, trials // 20)))
    print(f"{ok}/{max(1, trials // 20)} large-shape binning trials passed")
    ok = sum(loss_trial(ctx_, port_, seed0 + i) for i in range(trials))
    print(f"{ok}/{trials} loss trials passed (seeds {seed0}..{seed0 + trials - 1})")
