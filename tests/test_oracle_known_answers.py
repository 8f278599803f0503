"""Pins the CPU oracle (oracle/) against every known answer the reference's own tests hold for the
hot path, so that "GPU == oracle" means "GPU == reference".

Runs on CPU.  Each test runs against BOTH checkers when both are present: the plain-C
restatement (oracle/libdarbs_oracle.so, always) and the reference's own sources compiled here
(oracle/_ref/libdarbs_ref.so, built where /root/reference exists).  Citations are to the
reference's proj/tests/*.cpp.
"""
import math

import numpy as np
import pytest

from oracle.cpu import Scene

PRESETS = ["gaussian", "half-cosine-sq", "raised-cosine", "mod-sinc", "inv-multiquadratic"]
PI = math.pi


def one(o, k, dm2):
    st, w, dw = o.eval(k, [dm2])
    assert st == 0
    return float(w[0]), float(dw[0])


# ------------------------------------------------------------------------------------ kernel
def test_make_kernel_rejects_bad_parameters(any_oracle):
    """test_kernel.cpp:17-24."""
    o = any_oracle
    assert o.make_kernel("gaussian", 0.0, 1.0)[0] == 1
    assert o.make_kernel("gaussian", -1.0, 1.0)[0] == 1
    assert o.make_kernel("gaussian", 2.0, 0.0)[0] == 1
    assert o.make_kernel("gaussian", 2.0, -3.0)[0] == 1
    assert o.make_kernel("half-cosine-sq", 2.0, 1.0, 0)[0] == 1
    assert o.make_kernel("gaussian", 2.0, 1.0)[0] == 0


def test_cutoffs_per_family(any_oracle):
    """test_kernel.cpp:26-38."""
    o = any_oracle
    assert o.make_kernel("half-cosine-sq", 2.0, 18.0 / PI)[1].cutoff == pytest.approx(9.0, rel=1e-12)
    assert o.make_kernel("raised-cosine", 1.0, 2.5 / PI)[1].cutoff == pytest.approx(6.25, rel=1e-12)
    assert o.make_kernel("mod-sinc", 1.0, 3.0 / PI)[1].cutoff == pytest.approx(9.0, rel=1e-12)
    g = o.make_kernel("gaussian", 2.0, 1.0)[1]
    assert g.unbounded and g.cutoff == pytest.approx(9.0)
    assert o.make_kernel("inv-multiquadratic", 2.0, 1.0)[1].unbounded


def test_eval_reference_values(any_oracle):
    """test_kernel.cpp:40-57."""
    o = any_oracle
    hc = o.make_kernel("half-cosine-sq", 2.0, 18.0 / PI)[1]
    assert one(o, hc, 0.0)[0] == pytest.approx(1.0, rel=1e-15)
    assert abs(one(o, hc, 9.0)[0]) < 1e-12
    g1 = o.make_kernel("gaussian", 2.0, 1.0)[1]
    assert one(o, g1, 1.0)[0] == pytest.approx(math.exp(-1.0), rel=1e-15)
    ms = o.make_kernel("mod-sinc", 1.0, 3.0 / PI)[1]
    assert one(o, ms, 0.0)[0] == pytest.approx(1.0, rel=1e-12)
    rc = o.make_kernel("raised-cosine", 1.0, 2.5 / PI)[1]
    assert one(o, rc, 0.0)[0] == pytest.approx(1.0, rel=1e-15)
    assert abs(one(o, rc, 6.25)[0]) < 1e-12
    iq = o.make_kernel("inv-multiquadratic", 2.0, 1.0)[1]
    assert one(o, iq, 3.0)[0] == pytest.approx(0.5, rel=1e-15)


def test_gaussian_xi1_is_exp_bitwise(any_oracle):
    """test_kernel.cpp:59-64 (machine precision, compared with ==)."""
    g = any_oracle.make_kernel("gaussian", 2.0, 1.0)[1]
    for dm2 in (0.0, 0.3, 1.0, 2.5, 8.9):
        assert one(any_oracle, g, dm2)[0] == math.exp(-dm2)


def test_eval_rejects_invalid_dm2(any_oracle):
    """test_kernel.cpp:66-71."""
    g = any_oracle.preset("gaussian")
    for bad in (-0.1, float("nan"), float("inf")):
        assert any_oracle.eval(g, [bad])[0] == 1


@pytest.mark.parametrize("name", PRESETS)
def test_weight_range_center_cutoff_monotone(any_oracle, name):
    """test_kernel.cpp:73-87 (range, w(0)=1, zero past the cutoff), :89-101 (monotone decay),
    :103-108 (exact zero at the cutoff of the cosine families)."""
    o = any_oracle
    k = o.preset(name)
    assert one(o, k, 0.0)[0] == pytest.approx(1.0, rel=1e-12)
    rng = np.random.default_rng(11)
    dm2 = rng.uniform(0.0, k.cutoff * 1.5, 2000)
    _, w, _ = o.eval(k, dm2)
    assert w.min() >= 0.0 and w.max() <= 1.0
    assert np.all(w[dm2 > k.cutoff] == 0.0)
    grid = k.cutoff * np.arange(0, 401) / 400.0
    _, wg, _ = o.eval(k, grid)
    assert np.all(np.diff(wg) <= 1e-12)
    if name in ("half-cosine-sq", "raised-cosine"):
        assert abs(one(o, k, k.cutoff)[0]) < 1e-12


@pytest.mark.parametrize("name", PRESETS)
def test_analytic_derivative_matches_finite_differences(any_oracle, name):
    """test_kernel.cpp:110-116 (grad_check_kernel < 1e-4): central differences, away from the cutoff
    and (mod-sinc) from the kinks of |sin|."""
    o = any_oracle
    k = o.preset(name)
    rng = np.random.default_rng(5)
    dm2 = rng.uniform(0.05, 0.9 * k.cutoff, 1000)
    h = 1e-5
    _, wp, _ = o.eval(k, dm2 + h)
    _, wm, _ = o.eval(k, dm2 - h)
    _, _, dw = o.eval(k, dm2)
    fd = (wp - wm) / (2 * h)
    err = np.abs(fd - dw) / np.maximum(np.maximum(np.abs(fd), np.abs(dw)), 1e-4)
    if name == "mod-sinc":
        u = np.sqrt(dm2) / k.xi
        err = err[np.abs(np.sin(u)) > 1e-3]
    assert err.max() < 1e-4


def test_presets_and_psi_table(any_oracle):
    """kernel.cpp:223-240 presets; psi_table.hpp:20-26 frozen correction factors."""
    o = any_oracle
    want = {"gaussian": (0, 2.0, 2.0, 9.0, 1.0), "half-cosine-sq": (1, 2.0, 18.0 / PI, 9.0, 1.36),
            "raised-cosine": (2, 1.0, 2.5 / PI, 6.25, 0.6552), "mod-sinc": (3, 1.0, 3.0 / PI, 9.0, 1.1762),
            "inv-multiquadratic": (4, 2.0, 1.0, 9.0, 1.6054)}
    for name, (fam, beta, xi, cut, psi) in want.items():
        k = o.preset(name)
        assert (k.family, k.beta, k.lobes) == (fam, beta, 1)
        assert k.xi == pytest.approx(xi, rel=1e-15)
        assert k.cutoff == pytest.approx(cut, rel=1e-12)
        assert o.default_psi(name) == psi
    assert o.default_psi("nope") < 0


# ---------------------------------------------------------------------------------- geometry
def test_conic_and_radius_known_answers(any_oracle):
    """test_geometry.cpp:181-197: radius 3 / 3 / 6, non-PD throws degenerate_covariance."""
    o = any_oracle
    hc = o.make_kernel("half-cosine-sq", 2.0, 18.0 / PI)[1]
    g = o.preset("gaussian")
    assert o.conic_and_radius(hc, [[1, 0, 1]])[2][0] == pytest.approx(3.0)
    assert o.conic_and_radius(g, [[1, 0, 1]])[2][0] == pytest.approx(3.0)
    assert o.conic_and_radius(g, [[4, 0, 1]])[2][0] == pytest.approx(6.0)
    assert o.conic_and_radius(g, [[1, 2, 1]])[0] == 2


def test_conic_inverts_covariance_and_eigenvalues(any_oracle):
    """test_geometry.cpp:199-220: conic * cov = I to 1e-9; eigenvalues vs an independent solver 1e-10."""
    o = any_oracle
    g = o.preset("gaussian")
    rng = np.random.default_rng(31)
    a = rng.uniform(0.5, 9.0, 100)
    c = rng.uniform(0.5, 9.0, 100)
    b = rng.uniform(-0.9, 0.9, 100) * np.sqrt(a * c)
    st, conic, radius, lam = o.conic_and_radius(g, np.stack([a, b, c], 1))
    assert st == 0
    for i in range(100):
        cov = np.array([[a[i], b[i]], [b[i], c[i]]])
        con = np.array([[conic[i, 0], conic[i, 1]], [conic[i, 1], conic[i, 2]]])
        assert np.abs(con @ cov - np.eye(2)).max() < 1e-9
        ev = np.linalg.eigvalsh(cov)
        assert np.abs(np.sort(lam[i]) - ev).max() < 1e-10
        assert radius[i] == math.ceil(3.0 * math.sqrt(ev[1]))


IDENTITY_CAMERA = np.array([100, 100, 50, 50, 100, 100, 1, 0, 0, 0, 0, 1, 0, 0, 0, 0, 1, 0, 0, 0, 0, 1.0])


def test_full_projection_of_a_primitive(any_oracle):
    """test_geometry.cpp:298-314: mu2.x = 50, depth 2, cov2 = 25.3 I, conic.a = 1/25.3; behind the
    camera -> culled.  Also psi + dilation 1.36 -> 1.66 (:161-166) through a unit-covariance splat."""
    o = any_oracle
    g = o.preset("gaussian")
    prim = np.array([[0, 0, 2, 0.1, 0.1, 0.1, 1, 0, 0, 0, 1, 1, 1, 1.0]])
    st, p = o.project(g, 1.0, prim, IDENTITY_CAMERA)
    assert st == 0 and p["valid"][0] == 1
    assert p["mu2"][0, 0] == pytest.approx(50.0)
    assert p["depth"][0] == pytest.approx(2.0)
    assert p["cov2"][0, 0] == pytest.approx(25.3, rel=1e-9)
    assert p["conic"][0, 0] == pytest.approx(1.0 / 25.3, rel=1e-9)
    prim[0, 2] = -2.0
    assert o.project(g, 1.0, prim, IDENTITY_CAMERA)[1]["valid"][0] == 0
    # scale 0.02 at z = 2 with f = 100 projects to unit covariance: psi 1.36 + 0.3 -> 1.66
    prim = np.array([[0, 0, 2, 0.02, 0.02, 0.02, 1, 0, 0, 0, 1, 1, 1, 1.0]])
    st, p = o.project(g, 1.36, prim, IDENTITY_CAMERA)
    assert p["cov2"][0, 0] == pytest.approx(1.66, rel=1e-12)
    assert p["cov2"][0, 2] == pytest.approx(1.66, rel=1e-12)
    # error taxonomy: psi <= 0 and scale <= 0 are invalid_parameter (test_geometry.cpp:71-72,:177-178)
    assert o.project(g, 0.0, prim, IDENTITY_CAMERA)[0] == 1
    prim[0, 3] = 0.0
    assert o.project(g, 1.0, prim, IDENTITY_CAMERA)[0] == 1


def test_backward_projection_zero_linear_and_finite_differences(any_oracle):
    """test_geometry.cpp:222-296: zero upstream -> zero; linear in psi; FD rel < 1e-3 (the FD runs on
    the scalar L = <G, cov2_raw(psi=1, dilation=0)> + <g, mu2>)."""
    o = any_oracle
    g = o.preset("gaussian")
    rng = np.random.default_rng(7)
    cam = IDENTITY_CAMERA.copy()
    n = 20
    prims = np.zeros((n, 14))
    prims[:, 0:2] = rng.uniform(-0.5, 0.5, (n, 2))
    prims[:, 2] = rng.uniform(3.0, 5.0, n)
    prims[:, 3:6] = rng.uniform(0.2, 0.9, (n, 3))
    prims[:, 6:10] = rng.normal(size=(n, 4))
    prims[:, 10:14] = 0.5
    gc = rng.normal(size=(n, 4))
    gc[:, 2] = gc[:, 1]  # symmetric upstream
    gm = rng.normal(size=(n, 2))
    z = o.backward_projection(1.0, np.zeros((n, 4)), np.zeros((n, 2)), prims, cam)
    assert all(np.all(a == 0.0) for a in z)
    g1 = o.backward_projection(1.0, gc, np.zeros((n, 2)), prims, cam)
    g2 = o.backward_projection(2.0, gc, np.zeros((n, 2)), prims, cam)
    for a, b in zip(g1, g2):
        assert np.abs(b - 2 * a).max() <= 1e-12 * max(1.0, np.abs(b).max())

    def scalar(p):
        st, pr = o.project(g, 1.0, p, cam, dilation=0.0)
        assert st == 0
        cov = pr["cov2"]
        return (gc[:, 0] * cov[:, 0] + (gc[:, 1] + gc[:, 2]) * cov[:, 1] + gc[:, 3] * cov[:, 2]
                + (gm * pr["mu2"]).sum(1))

    d_mu, d_scale, d_rot = o.backward_projection(1.0, gc, gm, prims, cam)
    analytic = np.concatenate([d_mu, d_scale, d_rot], axis=1)
    h = 1e-6
    for col in range(10):
        pp, pm = prims.copy(), prims.copy()
        pp[:, col] += h
        pm[:, col] -= h
        fd = (scalar(pp) - scalar(pm)) / (2 * h)
        an = analytic[:, col]
        err = np.abs(fd - an) / np.maximum(np.maximum(np.abs(fd), np.abs(an)), 1e-4)
        assert err.max() < 1e-3, (col, err.max())


# -------------------------------------------------------------------------------- rasterizer
def splat(o, k, mu, cov, depth, opacity, color):
    """make_splat of test_rasterizer.cpp:16-24."""
    st, conic, radius, _ = o.conic_and_radius(k, [cov])
    assert st == 0
    return dict(mu2=mu, cov2=cov, conic=conic[0], radius=radius[0], depth=depth, opacity=opacity, rgb=color)


def scene_of(splats):
    if not splats:
        return Scene(np.zeros((0, 2)), np.zeros((0, 3)), np.zeros((0, 3)), np.zeros(0), np.zeros(0), np.zeros(0),
                     np.zeros((0, 3)))
    return Scene(*[np.array([s[key] for s in splats], dtype=np.float64)
                   for key in ("mu2", "cov2", "conic", "radius", "depth", "opacity", "rgb")])


def lists_of(offsets, plist):
    return [plist[offsets[t]:offsets[t + 1]].tolist() for t in range(offsets.size - 1)]


def test_binning_membership_and_ordering(any_oracle):
    """test_rasterizer.cpp:59-82."""
    o = any_oracle
    g = o.preset("gaussian")
    a = splat(o, g, (8, 8), (0.4, 0, 0.4), 1.0, 0.9, (1, 1, 1))
    offsets, plist, _ = o.bin(scene_of([a]), 32, 32)
    assert [len(x) for x in lists_of(offsets, plist)] == [1, 0, 0, 0]
    b = splat(o, g, (16, 16), (400.0, 0, 400.0), 0.5, 0.9, (1, 1, 1))
    offsets, plist, _ = o.bin(scene_of([a, b]), 32, 32)
    lists = lists_of(offsets, plist)
    assert all(1 in x for x in lists)
    assert lists[0][0] == 1 and lists[0][-1] == 0  # depth ascending inside a tile


def test_equal_depths_ordered_by_index(any_oracle):
    """test_rasterizer.cpp:84-94."""
    o = any_oracle
    g = o.preset("gaussian")
    s = [splat(o, g, (8, 8), (1, 0, 1), 2.0, 0.5, (1, 1, 1)) for _ in range(4)]
    offsets, plist, _ = o.bin(scene_of(s), 16, 16)
    assert lists_of(offsets, plist)[0] == [0, 1, 2, 3]


def test_forward_basics(any_oracle):
    """test_rasterizer.cpp:96-130: empty scene, alpha clamp, closed-form single-splat blend (1e-12)."""
    o = any_oracle
    g = o.preset("gaussian")
    r = o.forward(g, scene_of([]), 8, 8, (0.2, 0.2, 0.2))
    assert np.allclose(r["image"], 0.2) and np.all(r["t_final"] == 1.0)
    s = splat(o, g, (4.5, 4.5), (1, 0, 1), 1.0, 1.0, (1, 0, 0))
    r = o.forward(g, scene_of([s]), 8, 8, (0, 0, 0))
    assert r["image"][4, 4, 0] == pytest.approx(0.99)
    assert r["image"][4, 4, 1] == pytest.approx(0.0)
    assert r["t_final"][4, 4] == pytest.approx(0.01)
    s = splat(o, g, (4.5, 4.5), (4, 0, 4), 1.0, 0.6, (0.3, 0.9, 0.1))
    bg = (0.2, 0.1, 0.4)
    r = o.forward(g, scene_of([s]), 8, 8, bg)
    for y in range(8):
        for x in range(8):
            dm2 = ((x - 4.0) ** 2 + (y - 4.0) ** 2) / 4.0
            w = 0.0 if dm2 > g.cutoff else math.exp(-dm2 / 2.0)
            alpha = min(0.99, 0.6 * w)
            if alpha < 1.0 / 255.0:
                alpha = 0.0
            for c in range(3):
                assert r["image"][y, x, c] == pytest.approx(s["rgb"][c] * alpha + bg[c] * (1 - alpha), rel=1e-12)


@pytest.mark.parametrize("name", ["gaussian", "raised-cosine", "half-cosine-sq"])
def test_tiled_equals_bruteforce(any_oracle, name):
    """test_rasterizer.cpp:140-155 / acceptance.cpp:356-372: tiled forward == brute-force oracle < 1e-6."""
    o = any_oracle
    k = o.preset(name)
    for seed in range(5):
        s = o.random_scene(k, 200, 64, 64, seed, round_f32=False)
        a = o.forward(k, s, 64, 64, (0.1, 0.2, 0.3))["image"]
        b = o.oracle_forward(k, s, 64, 64, (0.1, 0.2, 0.3))
        assert np.abs(a - b).max() < 1e-6


def test_output_channels_in_unit_range(any_oracle):
    """test_rasterizer.cpp:157-165 (mod-sinc)."""
    o = any_oracle
    k = o.preset("mod-sinc")
    s = o.random_scene(k, 300, 64, 64, 3, round_f32=False)
    img = o.forward(k, s, 64, 64, (0.1, 0.2, 0.3))["image"]
    assert img.min() >= 0.0 and img.max() <= 1.0 + 1e-12


def test_thread_count_independence_bitwise(any_oracle):
    """test_rasterizer.cpp:167-174 (forward) and :260-273 (backward)."""
    o = any_oracle
    k = o.preset("raised-cosine")
    s = o.random_scene(k, 300, 64, 64, 1, round_f32=False)
    g = o.random_image_grad(64, 64, 99, round_f32=False)
    outs = []
    for threads in (1, 4):
        fr = o.forward(k, s, 64, 64, (0.1, 0.2, 0.3), threads=threads, keep=True)
        st, grads = o.backward(fr["handle"], k, g, s, threads=threads)
        o.forward_free(fr["handle"])
        assert st == 0
        outs.append((fr["image"], fr["processed"], grads))
    assert np.array_equal(outs[0][0], outs[1][0])
    assert np.array_equal(outs[0][1], outs[1][1])
    assert np.array_equal(outs[0][2], outs[1][2])


def test_backward_contract_and_zero_upstream(any_oracle):
    """test_rasterizer.cpp:176-185 (aux mismatch -> contract_violation), :187-197 (zero upstream)."""
    o = any_oracle
    k = o.preset("gaussian")
    s = o.random_scene(k, 50, 32, 32, 2, round_f32=False)
    fr = o.forward(k, s, 32, 32, (0, 0, 0), keep=True)
    assert o.backward(fr["handle"], k, np.zeros((16, 32, 3)), s)[0] == 4
    assert o.backward(fr["handle"], k, np.zeros((32, 32, 3)), s.take(np.arange(49)))[0] == 4
    st, grads = o.backward(fr["handle"], k, np.zeros((32, 32, 3)), s)
    o.forward_free(fr["handle"])
    assert st == 0 and np.all(grads == 0.0)


def test_rasterizer_gradients_match_finite_differences(any_oracle):
    """test_rasterizer.cpp:220-258 / acceptance.cpp:262-314: all 9 gradient components, raised-cosine,
    rel < 1e-3 with denominator floor 1e-4, FD on L = <g, image>."""
    o = any_oracle
    k = o.preset("raised-cosine")
    w, h, n = 20, 18, 18
    s = o.random_scene(k, n, w, h, 31, round_f32=False)
    g = o.random_image_grad(w, h, 99, round_f32=False)
    bg = (0.1, 0.2, 0.3)
    fr = o.forward(k, s, w, h, bg, keep=True)
    st, grads = o.backward(fr["handle"], k, g, s)
    o.forward_free(fr["handle"])
    assert st == 0

    def loss(sc):
        return float((o.forward(k, sc, w, h, bg)["image"] * g).sum())

    fields = [("rgb", 0), ("rgb", 1), ("rgb", 2), ("opacity", None), ("conic", 0), ("conic", 1), ("conic", 2),
              ("mu2", 0), ("mu2", 1)]
    hstep = 1e-6
    worst = 0.0
    for comp, (field, col) in enumerate(fields):
        for i in range(n):
            def bump(delta):
                sc = s.take(np.arange(n))
                arr = getattr(sc, field)
                if col is None:
                    arr[i] += delta
                else:
                    arr[i, col] += delta
                return loss(sc)
            fd = (bump(hstep) - bump(-hstep)) / (2 * hstep)
            an = grads[i, comp]
            worst = max(worst, abs(fd - an) / max(abs(fd), abs(an), 1e-4))
    assert worst < 1e-3, worst


def test_adam_known_answers(any_oracle):
    """test_loss.cpp:84-115: zero gradient is a no-op, first step ~ -lr, constant-gradient limit, shape
    mismatch is a contract violation (checked at the C ABI; the oracle takes one dim)."""
    o = any_oracle
    p0 = np.array([1.0, -2.0, 3.0])
    lrs = np.array([0.1, 0.01, 0.001])
    st, p, m, v = o.adam_step(p0, np.zeros(3), np.zeros(3), np.zeros(3), lrs, 1)
    assert st == 0 and np.array_equal(p, p0)
    st, p, m, v = o.adam_step(p0, np.array([0.5, -0.25, 4.0]), np.zeros(3), np.zeros(3), lrs, 1)
    assert np.allclose(p - p0, -lrs * np.array([1, -1, 1]), rtol=1e-6)
    p, m, v = p0.copy(), np.zeros(3), np.zeros(3)
    for t in range(1, 201):
        st, p, m, v = o.adam_step(p, np.array([2.0, 2.0, 2.0]), m, v, lrs, t)
    assert np.allclose(p - p0, -200 * lrs, rtol=1e-6)


# ------------------------------------------------------------------ restatement == reference
# ------------------------------------------------------------------ loss (tests/test_loss.cpp:23-82)
def test_loss_identical_images(any_oracle):
    """test_loss.cpp:23-34"""
    o = any_oracle
    x = o.random_image(16, 16, 1, round_f32=False)
    st, s = o.ssim(x, x)
    assert st == 0 and s == pytest.approx(1.0, rel=1e-12)
    for lam in (0.0, 0.2, 1.0):
        st, (total, l1, dssim), grad = o.loss_total(x, x, lam)
        assert st == 0
        assert abs(total) <= 1e-12 and l1 == 0.0 and abs(dssim) <= 1e-12
        assert np.abs(grad).max() < 1e-12


def test_loss_pure_l1_on_constant_offset(any_oracle):
    """test_loss.cpp:36-45"""
    o = any_oracle
    x = np.minimum(o.random_image(12, 12, 2, round_f32=False), 0.8)
    st, (total, l1, dssim), _ = o.loss_total(x + 0.1, x, 0.0)
    assert total == pytest.approx(0.1, rel=1e-12) and l1 == pytest.approx(0.1, rel=1e-12)


def test_loss_gradient_matches_finite_differences(any_oracle):
    """test_loss.cpp:53-77: central differences, step 1e-6, every 7th value, rel < 1e-3."""
    o = any_oracle
    w, h = 10, 9
    x = o.random_image(w, h, 3, round_f32=False)
    y = o.random_image(w, h, 4, round_f32=False)
    for lam in (0.2, 1.0):
        st, _, grad = o.loss_total(x, y, lam)
        worst = 0.0
        flat = grad.reshape(-1)
        for i in range(0, x.size, 7):
            hi, lo = x.copy().reshape(-1), x.copy().reshape(-1)
            hi[i] += 1e-6
            lo[i] -= 1e-6
            fd = (o.loss_total(hi.reshape(x.shape), y, lam, want_grad=False)[1][0] -
                  o.loss_total(lo.reshape(x.shape), y, lam, want_grad=False)[1][0]) / 2e-6
            worst = max(worst, abs(fd - flat[i]) / max(abs(fd), abs(flat[i]), 1e-8))
        assert worst < 1e-3


def test_loss_mixes_linearly_in_lambda(any_oracle):
    """test_loss.cpp:79-86"""
    o = any_oracle
    x = o.random_image(14, 14, 5, round_f32=False)
    y = o.random_image(14, 14, 6, round_f32=False)
    l0 = o.loss_total(x, y, 0.0)[1]
    l1 = o.loss_total(x, y, 1.0)[1]
    mid = o.loss_total(x, y, 0.3)[1]
    assert mid[0] == pytest.approx(0.7 * l0[1] + 0.3 * l1[2], rel=1e-12)


@pytest.mark.parametrize("size", [(1, 1), (3, 4), (10, 9), (37, 21), (64, 48)])
def test_port_loss_matches_reference_sources(port, ref, size):
    w, h = size
    x, y = port.random_image(w, h, 11), port.random_image(w, h, 12)
    assert np.array_equal(x, ref.random_image(w, h, 11))
    for lam in (0.0, 0.2, 1.0):
        _, a, ga = port.loss_total(x, y, lam)
        _, b, gb = ref.loss_total(x, y, lam)
        # (1x1: every tap folds onto the one pixel, b2 = C2 exactly up to rounding -> 1e-14 noise)
        assert np.abs(np.array(a) - np.array(b)).max() <= 1e-12
        assert np.abs(ga - gb).max() <= 1e-12 * max(1.0, np.abs(gb).max())


@pytest.mark.parametrize("name", PRESETS)
def test_port_matches_reference_sources(port, ref, name):
    """The plain-C restatement against the reference's own sources on the same inputs: integer
    outputs identical, FP64 outputs to 1e-12 (same algorithm, possibly different libm call order)."""
    k = port.preset(name)
    kr = ref.preset(name)
    assert (k.family, k.beta, k.xi, k.lobes, k.cutoff, k.unbounded) == (
        kr.family, kr.beta, kr.xi, kr.lobes, kr.cutoff, kr.unbounded)
    w, h, n = 70, 50, 400
    s = port.random_scene(k, n, w, h, 4)
    sr = ref.random_scene(kr, n, w, h, 4)
    for f in ("mu2", "cov2", "conic", "radius", "depth", "opacity", "rgb"):
        assert np.array_equal(getattr(s, f), getattr(sr, f)), f
    for a, b in zip(port.bin(s, w, h), ref.bin(s, w, h)):
        assert np.array_equal(a, b)
    g = port.random_image_grad(w, h, 5)
    assert np.array_equal(g, ref.random_image_grad(w, h, 5))
    fa = port.forward(k, s, w, h, (0.1, 0.2, 0.3), threads=2, keep=True)
    fb = ref.forward(kr, s, w, h, (0.1, 0.2, 0.3), threads=2, keep=True)
    assert np.array_equal(fa["processed"], fb["processed"])
    assert np.array_equal(fa["contributors"], fb["contributors"])
    assert np.abs(fa["image"] - fb["image"]).max() <= 1e-12
    assert np.abs(fa["t_final"] - fb["t_final"]).max() <= 1e-12
    _, ga = port.backward(fa["handle"], k, g, s)
    _, gb = ref.backward(fb["handle"], kr, g, s)
    port.forward_free(fa["handle"])
    ref.forward_free(fb["handle"])
    assert np.abs(ga - gb).max() <= 1e-11 * max(1.0, np.abs(gb).max())
