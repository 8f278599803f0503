"""GPU parity of the per-primitive stages (kernel eval, project, backward_projection,
evaluate_view, adam) against the CPU oracle, through the C ABI.

Mirrors tests/test_kernel.cpp, tests/test_geometry.cpp and the Adam cases of
tests/test_loss.cpp of the reference (cited per test).

Tolerances:
  * kernel weight (FP32 fast path, MUFU approximations): |w - oracle| <= 2e-6 absolute,
    derivative 1e-5 relative-to-max; FP64 path 1e-6 (float32 output rounding);
  * projection outputs are computed in FP64 on the device and rounded to float32:
    relative 1e-6; radius and visibility exact;
  * backward_projection / parameter gradients: relative 1e-5 of the per-array max
    (FP64 chain, float32 outputs) resp. 1e-3 relative with a floor of 5e-4 of the largest
    gradient (5e-4) end to end (float32 accumulation in the render backward, see the test);
  * adam: float32 update against the FP64 reference, 1e-6 absolute on parameters.
"""
import numpy as np
import pytest

from conftest import f32, rel_err

pytestmark = pytest.mark.gpu

PRESETS = ["gaussian", "half-cosine-sq", "raised-cosine", "mod-sinc", "inv-multiquadratic"]

DEMO_CAMERA = np.array([80, 80, 32, 32, 64, 64,
                        -0.3894183423, 0, 0.921060994, 4.278389336e-17,
                        -0.2646649291, 0.9578262852, -0.1118985373, -1.14366835e-16,
                        -0.8822164303, -0.2873478856, -0.3729951242, 3.132091953,
                        0, 0, 0, 1.0])


def random_raw(n, seed, scale_lo=0.03, scale_hi=0.12, spread=0.6):
    rng = np.random.default_rng(seed)
    raw = np.zeros((n, 14))
    raw[:, 0:3] = rng.uniform(-spread, spread, (n, 3))
    raw[:, 3:6] = np.log(rng.uniform(scale_lo, scale_hi, (n, 3)))
    raw[:, 6:10] = rng.normal(size=(n, 4))
    raw[:, 10] = rng.normal(size=n)
    raw[:, 11:14] = rng.normal(size=(n, 3))
    return f32(raw)


@pytest.mark.parametrize("name", PRESETS)
def test_eval_matches_oracle(ctx, port, darbs, name):
    """test_kernel.cpp:40-57, :73-87, :103-108: values, range, zero past the cutoff."""
    k = port.preset(name)
    gk = darbs.kernel_preset(name)
    assert (gk.family, gk.beta, gk.xi, gk.lobes, gk.cutoff, gk.unbounded) == (
        k.family, k.beta, k.xi, k.lobes, k.cutoff, k.unbounded)
    dm2 = f32(np.concatenate([np.linspace(0.0, k.cutoff * 1.5, 4001), [0.0, k.cutoff, 1e-20]]))
    _, w_ref, dw_ref = port.eval(k, dm2.astype(np.float64))
    w, dw = ctx.eval(gk, dm2)
    assert np.abs(w - w_ref).max() <= 2e-6
    assert np.abs(dw - dw_ref).max() <= 1e-5 * max(1.0, np.abs(dw_ref).max())
    assert w.min() >= 0.0 and w.max() <= 1.0 + 1e-6
    assert np.all(w[dm2 > k.cutoff] == 0.0)
    wx, dwx = ctx.eval(gk, dm2, exact=True)
    assert np.abs(wx - w_ref).max() <= 1e-6
    assert np.abs(dwx - dw_ref).max() <= 1e-6 * max(1.0, np.abs(dw_ref).max())


def test_eval_generic_families(ctx, port, darbs):
    """Multi-lobe and non-preset beta go through the generic functor (test_kernel.cpp:153-161)."""
    for fam, beta, xi, lobes in [("raised-cosine", 1.0, 2.5 / np.pi, 2), ("gaussian", 1.0, 1.3, 1),
                                 ("half-cosine", 1.0, 1.7, 1), ("mod-sinc", 1.0, 3 / np.pi, 2)]:
        gk = darbs.make_kernel(fam, beta, xi, lobes)
        st, k = port.make_kernel(gk.family, beta, xi, lobes)
        assert st == 0 and gk.cutoff == pytest.approx(k.cutoff, rel=1e-15)
        dm2 = f32(np.linspace(1e-3, k.cutoff * 1.2, 2001))
        _, w_ref, dw_ref = port.eval(k, dm2.astype(np.float64))
        w, dw = ctx.eval(gk, dm2)
        assert np.abs(w - w_ref).max() <= 5e-6


def test_eval_rejects_invalid_dm2(ctx, darbs):
    """test_kernel.cpp:66-71."""
    gk = darbs.kernel_preset("gaussian")
    for bad in (-0.1, np.nan, np.inf):
        with pytest.raises(darbs.DarbsError) as e:
            ctx.eval(gk, f32([0.5, bad]))
        assert e.value.status == 1


@pytest.mark.parametrize("name", ["gaussian", "half-cosine-sq", "raised-cosine", "inv-multiquadratic"])
def test_project_matches_oracle(ctx, port, darbs, name):
    """project_primitive on random primitives through the demo camera (geometry.cpp:66-87)."""
    k = port.preset(name)
    psi = port.default_psi(name)
    raw = random_raw(500, 3)
    raw[7, 0:3] = (3.5288, 1.1492, 1.4920)  # behind the camera for the demo view
    prims_g = ctx.realize(raw)
    prims_o = port.realize(raw.astype(np.float64))
    assert np.abs(prims_g - prims_o).max() <= 2e-7 * np.abs(prims_o).max()
    # feed the SAME float32 primitives to both sides
    st, o = port.project(k, psi, prims_g.astype(np.float64), DEMO_CAMERA)
    assert st == 0
    g = ctx.project(darbs.kernel_preset(name), psi, prims_g, DEMO_CAMERA)
    assert np.array_equal(g["valid"], o["valid"])
    assert 0 < g["valid"].sum() <= 500
    v = o["valid"] == 1
    assert np.array_equal(g["radius"][v], o["radius"][v])
    for key in ("mu2", "cov2", "conic", "depth"):
        assert rel_err(g[key][v], o[key][v], 1e-3).max() <= 1e-6, key


def test_project_known_answers(ctx, darbs):
    """Full projection of a primitive, test_geometry.cpp:298-314: cov2 = 25.3 I, conic.a = 1/25.3."""
    cam = np.array([100, 100, 50, 50, 100, 100, 1, 0, 0, 0, 0, 1, 0, 0, 0, 0, 1, 0, 0, 0, 0, 1.0])
    prim = f32([[0, 0, 2, 0.1, 0.1, 0.1, 1, 0, 0, 0, 1, 1, 1, 1]])
    g = ctx.project(darbs.kernel_preset("gaussian"), 1.0, prim, cam)
    assert g["valid"][0] == 1
    assert g["mu2"][0, 0] == pytest.approx(50.0)
    assert g["depth"][0] == pytest.approx(2.0)
    assert g["cov2"][0, 0] == pytest.approx(25.3, rel=1e-6)
    assert g["conic"][0, 0] == pytest.approx(1.0 / 25.3, rel=1e-6)
    prim[0, 2] = -2.0
    assert ctx.project(darbs.kernel_preset("gaussian"), 1.0, prim, cam)["valid"][0] == 0


def test_project_error_taxonomy(ctx, darbs):
    """scale <= 0 -> invalid_parameter (geometry.cpp:10-12, test_geometry.cpp:71-72);
    psi <= 0 -> invalid_parameter (geometry.cpp:44-46, test_geometry.cpp:177-178)."""
    cam = np.array([100, 100, 50, 50, 100, 100, 1, 0, 0, 0, 0, 1, 0, 0, 0, 0, 1, 0, 0, 0, 0, 1.0])
    prim = f32([[0, 0, 2, 0.0, 0.1, 0.1, 1, 0, 0, 0, 1, 1, 1, 1]])
    with pytest.raises(darbs.DarbsError) as e:
        ctx.project(darbs.kernel_preset("gaussian"), 1.0, prim, cam)
    assert e.value.status == 1
    prim[0, 3] = 0.1
    with pytest.raises(darbs.DarbsError) as e:
        ctx.project(darbs.kernel_preset("gaussian"), 0.0, prim, cam)
    assert e.value.status == 1


def test_backward_projection_matches_oracle(ctx, port):
    """backward_projection, geometry.cpp:111-168 (the reference checks it against finite
    differences, test_geometry.cpp:241-296)."""
    raw = random_raw(400, 5)
    prims = ctx.realize(raw)
    rng = np.random.default_rng(1)
    gc = f32(rng.normal(size=(400, 4)))
    gm = f32(rng.normal(size=(400, 2)))
    ref = port.backward_projection(1.36, gc.astype(np.float64), gm.astype(np.float64), prims.astype(np.float64),
                                   DEMO_CAMERA)
    got = ctx.backward_projection(1.36, gc, gm, prims, DEMO_CAMERA)
    for a, b in zip(got, ref):
        assert np.abs(a - b).max() <= 1e-5 * np.abs(b).max()
    # zero upstream -> zero (test_geometry.cpp:222-230); linear in psi (:232-245)
    z = ctx.backward_projection(1.36, np.zeros_like(gc), np.zeros_like(gm), prims, DEMO_CAMERA)
    assert all(np.all(a == 0.0) for a in z)
    g1 = ctx.backward_projection(1.0, gc, np.zeros_like(gm), prims, DEMO_CAMERA)
    g2 = ctx.backward_projection(2.0, gc, np.zeros_like(gm), prims, DEMO_CAMERA)
    for a, b in zip(g1, g2):
        assert np.abs(b - 2.0 * a).max() <= 1e-5 * np.abs(b).max()


@pytest.mark.parametrize("name", ["gaussian", "half-cosine-sq", "raised-cosine", "inv-multiquadratic"])
def test_evaluate_view_matches_oracle_chain(ctx, port, darbs, name):
    """One view of fit_scene's evaluate (fit3d.cpp:108-159) with a given dL/dimage: the GPU
    chain realize->project->forward->backward->param grads against the same chain built from the
    oracle's functions, fed the GPU's float32 splats at the rasterizer boundary."""
    k = port.preset(name)
    gk = darbs.kernel_preset(name)
    psi = port.default_psi(name)
    n = 600
    raw = random_raw(n, 9, scale_lo=0.02, scale_hi=0.08, spread=0.9)
    raw[3, 0:3] = (3.5288, 1.1492, 1.4920)  # culled primitive
    w = h = 64
    gimg = f32(port.random_image_grad(w, h, 77))
    pg = np.zeros((n, 14), np.float32)
    img = np.zeros((h, w, 3), np.float32)
    ctx.evaluate_view(gk, psi, raw, DEMO_CAMERA, (0, 0, 0), grad_image=gimg, param_grads=pg, image_out=img)

    prims = port.realize(raw.astype(np.float64))
    st, pr = port.project(k, psi, prims, DEMO_CAMERA)
    assert st == 0
    vis = np.flatnonzero(pr["valid"])
    assert vis.size < n
    from oracle.cpu import Scene

    s = Scene(pr["mu2"][vis], None, pr["conic"][vis], pr["radius"][vis], pr["depth"][vis], prims[vis, 10],
              prims[vis, 11:14])
    fr = port.forward(k, s, w, h, (0, 0, 0), threads=0, keep=True)
    st, sg = port.backward(fr["handle"], k, gimg.astype(np.float64), s, threads=0)
    port.forward_free(fr["handle"])
    ref = port.param_grads(psi, vis.astype(np.int32), sg, s.conic, s.opacity, s.rgb, prims, DEMO_CAMERA)
    assert np.abs(img - fr["image"]).max() <= 5e-5
    # floor: 5e-4 of the largest gradient, i.e. an absolute error of 5e-7 * max|ref| -- eight
    # float32 ulps of the largest partial sum.  scratch/diag_chain.py splits the error: all of it is
    # the float32 accumulation of the render backward (splat gradients differ by ~5e-7 absolute and
    # the chain multiplies d_mu2 by fx / z ~ 26); the FP32 preprocess-backward chain adds < 8e-5.
    err = rel_err(pg, ref, 5e-4 * max(1.0, np.abs(ref).max()))
    assert err.max() <= 1e-3, f"{err.max():.3e} at {np.unravel_index(err.argmax(), err.shape)}"
    assert np.all(pg[3] == 0.0)

    # accumulation over views is a plain += (fit3d.cpp:148-158)
    pg2 = pg.copy()
    ctx.evaluate_view(gk, psi, raw, DEMO_CAMERA, (0, 0, 0), grad_image=gimg, param_grads=pg2)
    # (two launches of an atomically accumulated sum: equal up to float32 summation order)
    assert rel_err(pg2, 2.0 * pg.astype(np.float64), 5e-4 * max(1.0, np.abs(ref).max())).max() <= 1e-3


def test_evaluate_view_overwrite_mode(ctx, darbs):
    """accumulate=False: the view overwrites param_grads (zeros for culled primitives), exactly
    what a zero fill followed by "+=" gives (fit3d.cpp:107, :148-158)."""
    gk = darbs.kernel_preset("raised-cosine")
    psi = darbs.default_psi("raised-cosine")
    n, w, h = 300, 64, 64
    raw = random_raw(n, 8)
    raw[7, 0:3] = (3.5288, 1.1492, 1.4920)  # behind the demo camera
    gimg = f32(np.random.default_rng(3).normal(size=(h, w, 3)))
    ref = np.zeros((n, 14), np.float32)
    ctx.evaluate_view(gk, psi, raw, DEMO_CAMERA, (0, 0, 0), grad_image=gimg, param_grads=ref)
    got = np.full((n, 14), 7.0, np.float32)  # stale contents must not survive
    ctx.evaluate_view(gk, psi, raw, DEMO_CAMERA, (0, 0, 0), grad_image=gimg, param_grads=got, accumulate=False)
    assert np.all(got[7] == 0.0)
    assert rel_err(got, ref, 1e-4 * max(1.0, np.abs(ref).max())).max() <= 1e-3
    # the setting applies to one call only: the next one accumulates again
    ctx.evaluate_view(gk, psi, raw, DEMO_CAMERA, (0, 0, 0), grad_image=gimg, param_grads=got)
    assert rel_err(got, 2.0 * ref.astype(np.float64), 1e-4 * max(1.0, np.abs(ref).max())).max() <= 1e-3


def test_evaluate_view_l1_loss_and_errors(ctx, port, darbs):
    """L1 branch of loss_total (loss.cpp:183-188, lambda = 0) and the two numeric_error exits of
    evaluate (fit3d.cpp:117-119)."""
    gk = darbs.kernel_preset("gaussian")
    n, w, h = 300, 64, 64
    raw = random_raw(n, 4)
    img = np.zeros((h, w, 3), np.float32)
    ctx.evaluate_view(gk, 1.0, raw, DEMO_CAMERA, (0, 0, 0), grad_image=np.zeros((h, w, 3), np.float32),
                      image_out=img)
    target = np.clip(img + f32(np.random.default_rng(0).normal(scale=0.05, size=img.shape)), 0, 1)
    pg = np.zeros((n, 14), np.float32)
    total, l1, dssim, mse = ctx.evaluate_view(gk, 1.0, raw, DEMO_CAMERA, (0, 0, 0), target=target, lam=0.0,
                                              param_grads=pg)
    d = img.astype(np.float64) - target
    assert l1 == pytest.approx(np.abs(d).mean(), rel=1e-5)
    assert total == pytest.approx(l1)
    assert mse == pytest.approx((d * d).mean(), rel=1e-5)
    # same gradients as feeding sign(d)/n by hand
    pg_ref = np.zeros((n, 14), np.float32)
    ctx.evaluate_view(gk, 1.0, raw, DEMO_CAMERA, (0, 0, 0), grad_image=f32(np.sign(d) / d.size), param_grads=pg_ref)
    assert rel_err(pg, pg_ref, 1e-6).max() <= 1e-3
    # every primitive behind the camera -> numeric_error
    raw_behind = raw.copy()
    raw_behind[:, 0:3] = (3.5288, 1.1492, 1.4920)
    with pytest.raises(darbs.DarbsError) as e:
        ctx.evaluate_view(gk, 1.0, raw_behind, DEMO_CAMERA, (0, 0, 0), target=target, param_grads=pg)
    assert e.value.status == 2
    with pytest.raises(darbs.DarbsError) as e:
        ctx.evaluate_view(gk, 1.0, raw, DEMO_CAMERA, (0, 0, 0), target=target, lam=1.5, param_grads=pg)
    assert e.value.status == 1


@pytest.mark.parametrize("lam", [0.2, 1.0])
def test_evaluate_view_dssim_loss(ctx, port, darbs, lam):
    """The full loss_total of fit_scene (loss.cpp:173-230, lambda = 0.2 by default,
    fit_common.hpp:16) inside evaluate_view: reported values against the oracle's loss on the
    rendered image, parameter gradients against the same view driven by the oracle's dL/dimage."""
    gk = darbs.kernel_preset("half-cosine-sq")
    psi = darbs.default_psi("half-cosine-sq")
    n, w, h = 300, 64, 64
    raw = random_raw(n, 5)
    img = np.zeros((h, w, 3), np.float32)
    ctx.evaluate_view(gk, psi, raw, DEMO_CAMERA, (0, 0, 0), grad_image=np.zeros((h, w, 3), np.float32),
                      image_out=img)
    target = np.clip(img + f32(np.random.default_rng(1).normal(scale=0.05, size=img.shape)), 0, 1)
    pg = np.zeros((n, 14), np.float32)
    total, l1, dssim, mse = ctx.evaluate_view(gk, psi, raw, DEMO_CAMERA, (0, 0, 0), target=target, lam=lam,
                                              param_grads=pg)
    st, (r_total, r_l1, r_dssim), r_grad = port.loss_total(img.astype(np.float64), target.astype(np.float64), lam)
    assert (total, l1, dssim) == pytest.approx((r_total, r_l1, r_dssim), abs=2e-6)
    pg_ref = np.zeros((n, 14), np.float32)
    ctx.evaluate_view(gk, psi, raw, DEMO_CAMERA, (0, 0, 0), grad_image=f32(r_grad), param_grads=pg_ref)
    assert rel_err(pg, pg_ref, 1e-3 * np.abs(pg_ref).max()).max() <= 2e-3


def test_adam_matches_oracle(ctx, port):
    """adam_step optim.hpp:24-39; zero-gradient no-op (test_loss.cpp:84-89), first step ~ -lr
    (:91-96)."""
    rng = np.random.default_rng(3)
    dim = 14 * 1000
    p0 = f32(rng.normal(size=dim))
    g = f32(rng.normal(size=dim))
    lrs = f32(rng.uniform(1e-4, 1e-2, size=dim))
    p, m, v = p0.copy(), np.zeros(dim, np.float32), np.zeros(dim, np.float32)
    pr, mr, vr = p0.astype(np.float64), np.zeros(dim), np.zeros(dim)
    for t in (1, 2, 3):
        ctx.adam_step(p, g, m, v, lrs, t)
        st, pr, mr, vr = port.adam_step(pr, g.astype(np.float64), mr, vr, lrs.astype(np.float64), t)
        assert np.abs(p - pr).max() <= 1e-6
        assert np.abs(m - mr).max() <= 1e-6 and np.abs(v - vr).max() <= 1e-6
    # first step moves every parameter by ~lr against the gradient sign
    p, m, v = p0.copy(), np.zeros(dim, np.float32), np.zeros(dim, np.float32)
    ctx.adam_step(p, g, m, v, lrs, 1)
    assert np.allclose(p - p0, -lrs * np.sign(g), rtol=1e-4, atol=3e-7)  # float32 ulp of |p| ~ 3
    # zero gradient is a no-op
    p, m, v = p0.copy(), np.zeros(dim, np.float32), np.zeros(dim, np.float32)
    ctx.adam_step(p, np.zeros(dim, np.float32), m, v, lrs, 1)
    assert np.array_equal(p, p0)


def test_entry_capacity_removes_the_wait_and_reports_overflow(darbs):
    """darbs_cuda_set_entry_capacity: with a capacity >= K the view is bit-identical to the default
    path (which waits for K); with a capacity below K nothing is written out of bounds, the view
    renders as if it were empty and the call that collects its loss reports contract_violation."""
    import torch

    from paper_2501_12369_b200 import synthetic as syn

    name, n, w, h = "raised-cosine", 40000, 320, 240
    gk, psi = darbs.kernel_preset(name), darbs.default_psi(name)
    truth = syn.scene_b(n, 1, half_extent=(1.0, 0.7, 0.7), scale_range=(0.004, 0.02))
    init = syn.perturb(truth, 2)
    cam = syn.orbit_camera(0, 1, w, h, 300.0)
    dev = torch.device("cuda", 0)
    with darbs.Context(0) as ctx:
        ctx.use_torch_stream()
        ctx.set_deterministic(True)
        target = torch.empty((h, w, 3), dtype=torch.float32, device=dev)
        ctx.evaluate_view(gk, psi, torch.from_numpy(truth).to(dev), cam, (0, 0, 0), grad_image=torch.zeros_like(target),
                          image_out=target)
        p = torch.from_numpy(init).to(dev)

        def run():
            g = torch.zeros((n, 14), device=dev)
            img = torch.empty_like(target)
            loss = ctx.evaluate_view(gk, psi, p, cam, (0, 0, 0), target=target, lam=0.2, param_grads=g, image_out=img,
                                     accumulate=False)
            return loss, g.cpu().numpy(), img.cpu().numpy()

        loss0, g0, img0 = run()
        k = ctx.work_counters()["entries"]
        assert k > 50000
        ctx.set_entry_capacity(int(1.25 * k))
        loss1, g1, img1 = run()
        assert ctx.work_counters()["entries"] == k
        assert loss1 == loss0 and np.array_equal(g1, g0) and np.array_equal(img1, img0)
        ctx.set_entry_capacity(k // 2)
        with pytest.raises(darbs.DarbsError) as e:
            run()
        assert e.value.status == 4 and "capacity" in str(e.value)
        ctx.set_entry_capacity(0)
        loss2, g2, img2 = run()
        assert loss2 == loss0 and np.array_equal(g2, g0)


def test_a_view_is_capturable_in_a_cuda_graph(darbs):
    """With an entry capacity nothing in darbs_cuda_evaluate_view synchronises with the host, so the
    whole view (preprocess ... parameter gradients) can be captured into
    a CUDA graph on the caller's stream and replayed: in the deterministic mode every replay is
    bit-identical to the eager call.  (A captured view reports neither loss nor status.)"""
    import torch

    from paper_2501_12369_b200 import synthetic as syn

    name, n, w, h = "half-cosine-sq", 30000, 256, 192
    gk, psi = darbs.kernel_preset(name), darbs.default_psi(name)
    truth = syn.scene_b(n, 1, half_extent=(1.0, 0.7, 0.7), scale_range=(0.004, 0.02))
    init = syn.perturb(truth, 2)
    cam = syn.orbit_camera(0, 1, w, h, 250.0)
    dev = torch.device("cuda", 0)
    stream = torch.cuda.Stream(dev)
    with torch.cuda.stream(stream), darbs.Context(0) as ctx:
        ctx.use_torch_stream()
        ctx.set_deterministic(True)
        target = torch.empty((h, w, 3), dtype=torch.float32, device=dev)
        ctx.evaluate_view(gk, psi, torch.from_numpy(truth).to(dev), cam, (0, 0, 0), grad_image=torch.zeros_like(target),
                          image_out=target)
        p = torch.from_numpy(init).to(dev)
        g = torch.zeros((n, 14), device=dev)
        img = torch.empty_like(target)

        def view(want_loss):
            return ctx.evaluate_view(gk, psi, p, cam, (0, 0, 0), target=target, lam=0.2, param_grads=g, image_out=img,
                                     accumulate=False, want_loss=want_loss)

        loss0 = view(True)
        g0, img0 = g.clone(), img.clone()
        ctx.set_entry_capacity(int(1.25 * ctx.work_counters()["entries"]))
        view(True)  # buffers sized by the capacity before the capture
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=stream):
            ctx.use_torch_stream()
            view(False)
        for _ in range(3):
            g.zero_()
            img.zero_()
            graph.replay()
            stream.synchronize()
            assert torch.equal(g, g0) and torch.equal(img, img0)
        ctx.set_entry_capacity(0)
        assert view(True) == loss0
