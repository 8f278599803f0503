"""GPU parity of bin / forward / backward against the CPU oracle, through the C ABI.

Mirrors the reference's tests/test_rasterizer.cpp (cited per test).  Inputs are
the reference's random_scene fixture rounded to float32, fed as
float32 to the GPU and widened to float64 for the oracle.

Tolerances (stated once, used everywhere):
  * tile ranges, point lists, sort keys, depth order, processed, contributors,
    skipped_nonfinite: bit-exact;
  * image, t_final: max |gpu - oracle| <= IMG_TOL = 2e-5 absolute (fp32 compositing
    of a few hundred terms in [0,1]);
  * splat gradients: |gpu - oracle| / max(|gpu|, |oracle|, floor_c) <= GRAD_TOL = 1e-3, the
    reference's own finite-difference criterion (test_rasterizer.cpp:242-243,257) with its
    denominator floor 1e-4 scaled by the size of the component over the scene:
    floor_c = max(1e-4, 1e-3 * max_i |oracle[i, c]|), i.e. an absolute error of 1e-6 of the
    component's scale S_c over the scene is always accepted.  A gradient component that is the
    cancelling sum of O(S) terms cannot be resolved below ~1e-7..1e-6 S in float32 (measured:
    the worst absolute error at 10k splats / 256x256 is 5.6e-6 on d_conic_b, S = 103).  On top of
    that, at least 99.9 % of all elements must meet the UNSCALED criterion (floor 1e-4).
"""
import numpy as np
import pytest

from conftest import f32, rel_err, scene_f32

pytestmark = pytest.mark.gpu

IMG_TOL = 2e-5
GRAD_TOL = 1e-3
GRAD_FLOOR = 1e-4
KERNELS = ["gaussian", "half-cosine-sq", "raised-cosine", "inv-multiquadratic", "mod-sinc"]
# (family, beta, xi, lobes) outside the presets: multi-lobe and other beta run the generic device
# path of the render kernels (kernel.cpp:73-104, tests/test_kernel.cpp:153-161)
GENERIC = ["custom:raised-cosine:1.0:0.6:2", "custom:half-cosine:1.0:1.9:1", "custom:mod-sinc:1.0:0.8:2",
           "custom:gaussian:1.5:2.0:1"]
BG = (0.1, 0.2, 0.3)


def gpu_kernel(darbs, name):
    return darbs.kernel_preset(name)


def oracle_keys(offsets, plist, order):
    rank = np.empty(order.size, dtype=np.int64)
    rank[order] = np.arange(order.size)
    tiles = np.repeat(np.arange(offsets.size - 1, dtype=np.uint64), np.diff(offsets))
    return (tiles << np.uint64(32)) | rank[plist].astype(np.uint64)


def check_bins(ctx, port, s, w, h):
    offsets, plist, order = port.bin(s, w, h)
    g = scene_f32(s)
    b = ctx.bin(g["mu2"], g["conic"], g["radius"], g["depth"], w, h)
    assert b["num_entries"] == plist.size
    assert np.array_equal(b["depth_order"], order)
    assert np.array_equal(b["point_list"], plist)
    lens = np.diff(offsets)
    nonempty = lens > 0
    assert np.array_equal(b["tile_ranges"][nonempty, 0], offsets[:-1][nonempty])
    assert np.array_equal(b["tile_ranges"][nonempty, 1], offsets[1:][nonempty])
    assert np.array_equal(b["tile_ranges"][~nonempty, 1] - b["tile_ranges"][~nonempty, 0], lens[~nonempty])
    assert np.array_equal(b["sort_keys"], oracle_keys(offsets, plist, order))


@pytest.mark.parametrize("name", ["gaussian", "raised-cosine"])
@pytest.mark.parametrize("shape", [(64, 64), (70, 50), (16, 16), (33, 97)])
@pytest.mark.parametrize("seed", [0, 1])
def test_bins_bit_exact(ctx, port, name, shape, seed):
    """bin_splats membership + depth order, test_rasterizer.cpp:59-82."""
    w, h = shape
    k = port.preset(name)
    s = port.random_scene(k, 500, w, h, seed)
    check_bins(ctx, port, s, w, h)


def test_bins_more_than_65536_tiles(ctx, port):
    """Beyond 65 536 tiles the tile sort switches from 16-bit to 32-bit keys (4208 x 4208 pixels =
    263 x 263 tiles); a few splats are made huge so that lists cross many tiles."""
    k = port.preset("gaussian")
    w = h = 4208
    s = port.random_scene(k, 3000, w, h, 5)
    s.radius[:8] = 900.0
    check_bins(ctx, port, s, w, h)


@pytest.mark.parametrize("shape,n", [((16, 400), 900), ((400, 16), 900), ((16, 16), 300), ((4112, 48), 4000),
                                     ((48, 4112), 4000), ((1920, 1080), 60000)])
def test_bins_every_digit_plan(ctx, port, shape, n):
    """The tile sort runs one radix pass per coordinate byte that can differ (binning.cu tile_plan): a
    single tile column or row drops that coordinate's pass, a single tile needs no pass, more than
    256 columns or rows switch to 32-bit keys with a second byte; the expand kernel's per-splat digit
    histograms take the byte-digit shortcut only for the two-pass 16-bit case.  Also a list long
    enough for several chunks of the 8192-pair passes and of the 2048-rank expand CTAs."""
    w, h = shape
    k = port.preset("half-cosine-sq")
    s = port.random_scene(k, n, w, h, 23)
    s.radius[:4] = 300.0  # a few splats across many tiles
    check_bins(ctx, port, s, w, h)


def test_bins_equal_depth_index_order(ctx, port):
    """Equal depths are ordered by splat index, test_rasterizer.cpp:84-94."""
    k = port.preset("gaussian")
    s = port.random_scene(k, 64, 32, 32, 5)
    s.depth[:] = 2.0
    s.depth[10:20] = 1.0
    check_bins(ctx, port, s, 32, 32)
    b = ctx.bin(f32(s.mu2), f32(s.conic), f32(s.radius), f32(s.depth), 32, 32)
    assert np.array_equal(b["depth_order"][:10], np.arange(10, 20))


def test_bins_huge_and_offscreen_and_nonfinite(ctx, port):
    """A huge splat lands in every tile (test_rasterizer.cpp:71-77); off-screen splats touch
    nothing; non-finite conic/radius are dropped and counted (rasterizer.cpp:39, :69-73)."""
    k = port.preset("gaussian")
    s = port.random_scene(k, 40, 64, 48, 7)
    s.radius[0] = 500.0
    s.mu2[1] = (-400.0, 10.0)
    s.mu2[2] = (30.0, 4000.0)
    s.conic[3, 1] = np.nan
    s.radius[4] = np.inf
    s.depth[5] = -3.0  # negative depth sorts first
    check_bins(ctx, port, s, 64, 48)
    g = scene_f32(s)
    out = ctx.forward(gpu_kernel_cached("gaussian"), **g, width=64, height=48, background=BG)
    ref = port.forward(k, s, 64, 48, BG)
    assert out["skipped"] == ref["skipped"] == 2
    assert np.array_equal(out["processed"], ref["processed"])
    assert np.array_equal(out["contributors"], ref["contributors"])


_KCACHE = {}


def custom_spec(name):
    _, family, beta, xi, lobes = name.split(":")
    return family, float(beta), float(xi), int(lobes)


def gpu_kernel_cached(name):
    import paper_2501_12369_b200 as d

    if name not in _KCACHE:
        _KCACHE[name] = d.make_kernel(*custom_spec(name)) if name.startswith("custom:") else d.kernel_preset(name)
    return _KCACHE[name]


def oracle_kernel(port, name):
    if not name.startswith("custom:"):
        return port.preset(name)
    family, beta, xi, lobes = custom_spec(name)
    st, k = port.make_kernel(gpu_kernel_cached(name).family, beta, xi, lobes)
    assert st == 0
    return k


def make_opaque(s, seed):
    """Opacities in [0.9, 1]: about one splat in five can reach the 0.99 alpha clamp
    (rasterizer.cpp:93, :202), so groups with and without such entries alternate in every stream."""
    rng = np.random.default_rng(seed)
    s.opacity[:] = f32(rng.uniform(0.9, 1.0, size=s.opacity.shape))
    s.opacity[::17] = 1.0
    return s


def run_forward_parity(ctx, port, name, n, w, h, seed, bg=BG, opaque=False):
    k = oracle_kernel(port, name)
    s = port.random_scene(k, n, w, h, seed)
    if opaque:
        make_opaque(s, seed)
    ref = port.forward(k, s, w, h, bg, threads=0)
    out = ctx.forward(gpu_kernel_cached(name), **scene_f32(s), width=w, height=h, background=bg)
    assert np.array_equal(out["processed"], ref["processed"]), "processed differs"
    assert np.array_equal(out["contributors"], ref["contributors"]), "contributors differ"
    assert np.abs(out["image"] - ref["image"]).max() <= IMG_TOL
    assert np.abs(out["t_final"] - ref["t_final"]).max() <= IMG_TOL
    return s, ref, out


@pytest.mark.parametrize("name", KERNELS)
@pytest.mark.parametrize("seed", [0, 1, 2])
def test_forward_parity_small(ctx, port, name, seed):
    """Tiled forward == the oracle's forward, 200 splats 64x64 (the sizes of
    test_rasterizer.cpp:140-155), every family."""
    run_forward_parity(ctx, port, name, 200, 64, 64, seed)


@pytest.mark.parametrize("name", ["gaussian", "half-cosine-sq", "raised-cosine"])
def test_forward_equals_bruteforce_oracle(ctx, port, name):
    """tiled == brute-force oracle_forward < 1e-6 in the reference (test_rasterizer.cpp:140-155);
    here the GPU image against oracle_forward within IMG_TOL."""
    k = port.preset(name)
    for seed in range(5):
        s = port.random_scene(k, 200, 64, 64, seed)
        brute = port.oracle_forward(k, s, 64, 64, BG)
        out = ctx.forward(gpu_kernel_cached(name), **scene_f32(s), width=64, height=64, background=BG, aux=False)
        assert np.abs(out["image"] - brute).max() <= IMG_TOL


@pytest.mark.parametrize("name", KERNELS + GENERIC)
def test_forward_parity_ragged_dense(ctx, port, name):
    """Image not a multiple of the tile size, lists longer than one 32-entry chunk, early
    termination on most pixels."""
    run_forward_parity(ctx, port, name, 3000, 77, 45, 11)


@pytest.mark.parametrize("name", KERNELS + GENERIC[:1])
def test_forward_parity_opaque(ctx, port, name):
    """Splats that reach the alpha clamp mixed with splats that cannot (the render kernels run
    a clamp-free variant on groups of entries whose opacity is below 0.98)."""
    run_forward_parity(ctx, port, name, 2500, 90, 70, 13, opaque=True)


@pytest.mark.parametrize("name", ["gaussian", "half-cosine-sq", "raised-cosine"])
def test_forward_and_backward_parity_needle_splats(ctx, port, name):
    """Ill-conditioned conics: sigma ~ 100 px along one axis against the 0.3 px^2 dilation
    floor along the other, at every angle.  In absolute pixel offsets the float32 quadratic form
    of such a needle carries an error far beyond the guard band, so the library takes their
    decisions in FP64 (splat.cuh kMaxKappa): processed / contributors stay the oracle's."""
    k = oracle_kernel(port, name)
    n, w, h = 400, 160, 128
    s = port.random_scene(k, n, w, h, 3)
    rng = np.random.default_rng(5)
    ang = rng.uniform(0, np.pi, n)
    s1 = rng.uniform(40.0, 120.0, n) ** 2
    s2 = np.full(n, 0.3) + rng.uniform(0.0, 0.5, n)
    needle = rng.uniform(size=n) < 0.5  # the other half stays well conditioned: both paths share streams
    c, sn = np.cos(ang), np.sin(ang)
    cov = np.stack([c * c * s1 + sn * sn * s2, c * sn * (s1 - s2), sn * sn * s1 + c * c * s2], axis=1)  # xx, xy, yy
    st, conic, radius, _lam = port.conic_and_radius(k, cov[needle])
    assert st == 0
    s.conic[needle] = f32(conic).astype(np.float64)  # float32-representable, as every parity input
    s.radius[needle] = radius
    s.opacity[needle] = f32(rng.uniform(0.05, 0.4, int(needle.sum())))
    g = port.random_image_grad(w, h, 9)
    fr = port.forward(k, s, w, h, BG, threads=0, keep=True)
    st, ref_g = port.backward(fr["handle"], k, g, s, threads=0)
    port.forward_free(fr["handle"])
    out = ctx.forward(gpu_kernel_cached(name), **scene_f32(s), width=w, height=h, background=BG)
    assert np.array_equal(out["processed"], fr["processed"])
    assert np.array_equal(out["contributors"], fr["contributors"])
    assert np.abs(out["image"] - fr["image"]).max() <= IMG_TOL
    got = ctx.backward(gpu_kernel_cached(name), f32(g), n)
    # decisions are exact, but the weight and its derivative still see the float32 quadratic form, whose
    # relative error grows with the eigenvalue ratio (~3 eps kappa, kappa up to 5e4 here): 5e-3 instead
    # of 1e-3 (measured: 1.4e-3 for the raised cosine, whose dw/dm ~ 1/sqrt(m); < 1e-3 for the others)
    assert grad_err(got, ref_g).max() <= 5.0 * GRAD_TOL


@pytest.mark.parametrize("name", ["gaussian", "half-cosine-sq", "inv-multiquadratic", "custom:raised-cosine:1.0:0.6:2"])
def test_results_do_not_depend_on_the_cull_segment(ctx, port, name):
    """The cull kernel may cover only the first entries of every tile's list; blocks whose pixels
    outlive them cull on inside the forward (render.cu forward_tail).  Whatever the segment, the
    per-pixel walk is the reference's (rasterizer.cpp:85-107): integer aux equal to the oracle's,
    images equal among themselves, gradients within tolerance."""
    k = oracle_kernel(port, name)
    n, w, h = 20000, 128, 96  # ~300 entries per tile
    s = port.random_scene(k, n, w, h, 17)
    s.opacity[:] = f32(np.random.default_rng(3).uniform(0.02, 0.3, n))  # slow saturation: long walks
    g = port.random_image_grad(w, h, 4)
    fr = port.forward(k, s, w, h, BG, threads=0, keep=True)
    st, ref_g = port.backward(fr["handle"], k, g, s, threads=0)
    port.forward_free(fr["handle"])
    sc = scene_f32(s)
    images = []
    try:
        for seg in (1 << 30, 8, 40, 96, 200):
            ctx.set_cull_segment(seg)
            out = ctx.forward(gpu_kernel_cached(name), **sc, width=w, height=h, background=BG)
            assert np.array_equal(out["processed"], fr["processed"]), seg
            assert np.array_equal(out["contributors"], fr["contributors"]), seg
            assert np.abs(out["image"] - fr["image"]).max() <= IMG_TOL
            images.append(out["image"].copy())
            got = ctx.backward(gpu_kernel_cached(name), f32(g), n)
            assert grad_err(got, ref_g).max() <= GRAD_TOL, seg
    finally:
        ctx.set_cull_segment(0)
    for img in images[1:]:
        assert np.abs(img - images[0]).max() <= 1e-6


def test_transmittance_floor_pixels_are_exact(ctx, port):
    """The last decision of a pixel, T < 1e-4 (rasterizer.cpp:100), cannot be taken in FP32 when T
    ends within a few 1e-9 of the floor: the forward kernel composites those pixels again in FP64
    (counted in work_counters().tfloor).  Dense scenes over several seeds so that the path runs."""
    flagged = 0
    for name in ("gaussian", "raised-cosine", "inv-multiquadratic"):
        for seed in (11, 12, 13):
            run_forward_parity(ctx, port, name, 3000, 77, 45, seed)
            flagged += ctx.work_counters()["tfloor"]
    assert flagged > 0


def test_forward_config1_bit_exact_counts(ctx, port):
    """BASELINE config 1: 10k splats, 256x256, half-cosine-squared."""
    s, ref, out = run_forward_parity(ctx, port, "half-cosine-sq", 10000, 256, 256, 0)
    wc = ctx.work_counters()
    assert wc["visits"] == int(ref["processed"].sum())
    assert wc["contributors"] == int(ref["contributors"].sum())


def test_forward_empty_scene_is_background(ctx, port):
    """test_rasterizer.cpp:98-102."""
    e = np.zeros((0,), dtype=np.float32)
    out = ctx.forward(gpu_kernel_cached("gaussian"), e.reshape(0, 2), e.reshape(0, 3), e, e, e, e.reshape(0, 3), 8, 8,
                      (0.2, 0.2, 0.2))
    assert np.allclose(out["image"], 0.2, atol=1e-7)
    assert np.all(out["t_final"] == 1.0)
    assert np.all(out["processed"] == 0) and np.all(out["contributors"] == 0)


def test_forward_alpha_clamp(ctx, port):
    """Opaque centred splat saturates at the alpha clamp, test_rasterizer.cpp:103-111."""
    k = port.preset("gaussian")
    st, conic, radius, _ = port.conic_and_radius(k, [[1.0, 0.0, 1.0]])
    out = ctx.forward(gpu_kernel_cached("gaussian"), f32([[4.5, 4.5]]), f32(conic), f32(radius), f32([1.0]), f32([1.0]),
                      f32([[1, 0, 0]]), 8, 8, (0, 0, 0))
    assert out["image"][4, 4, 0] == pytest.approx(0.99, abs=1e-6)
    assert out["image"][4, 4, 1] == 0.0
    assert out["t_final"][4, 4] == pytest.approx(0.01, abs=1e-6)


def test_forward_single_splat_closed_form(ctx, port):
    """Closed-form single-splat blend incl. cutoff and the 1/255 skip, test_rasterizer.cpp:112-130."""
    k = port.preset("gaussian")
    st, conic, radius, _ = port.conic_and_radius(k, [[4.0, 0.0, 4.0]])
    col, bg = np.array([0.3, 0.9, 0.1]), np.array([0.2, 0.1, 0.4])
    out = ctx.forward(gpu_kernel_cached("gaussian"), f32([[4.5, 4.5]]), f32(conic), f32(radius), f32([1.0]), f32([0.6]),
                      f32([col]), 8, 8, bg)
    for y in range(8):
        for x in range(8):
            dm2 = ((x + 0.5 - 4.5) ** 2 + (y + 0.5 - 4.5) ** 2) / 4.0
            w = 0.0 if dm2 > 9.0 else np.exp(-dm2 / 2.0)
            alpha = min(0.99, 0.6 * w)
            if alpha < 1.0 / 255.0:
                alpha = 0.0
            assert np.allclose(out["image"][y, x], col * alpha + bg * (1 - alpha), atol=2e-6)


def test_forward_output_in_unit_range(ctx, port):
    """Channels stay in [0,1] (mod-sinc), test_rasterizer.cpp:157-165."""
    k = port.preset("mod-sinc")
    s = port.random_scene(k, 150, 48, 48, 9)
    out = ctx.forward(gpu_kernel_cached("mod-sinc"), **scene_f32(s), width=48, height=48, background=(0.5, 0.5, 0.5))
    assert out["image"].min() >= 0.0 and out["image"].max() <= 1.0 + 1e-6


def test_forward_is_deterministic(ctx, port):
    """The reference is bitwise thread-count independent (test_rasterizer.cpp:167-174); the GPU
    forward has no atomics on its outputs and must be bitwise repeatable."""
    k = port.preset("gaussian")
    s = port.random_scene(k, 1000, 96, 64, 4)
    a = ctx.forward(gpu_kernel_cached("gaussian"), **scene_f32(s), width=96, height=64, background=(0, 0, 0))
    b = ctx.forward(gpu_kernel_cached("gaussian"), **scene_f32(s), width=96, height=64, background=(0, 0, 0))
    for key in ("image", "t_final", "processed", "contributors"):
        assert np.array_equal(a[key], b[key])


def grad_err(got, ref):
    floor = np.maximum(GRAD_FLOOR, 1e-3 * np.abs(ref).max(axis=0, keepdims=True))
    return rel_err(got, ref, floor)


def run_backward_parity(ctx, port, name, n, w, h, seed, gseed=32, opaque=False):
    k = oracle_kernel(port, name)
    s = port.random_scene(k, n, w, h, seed)
    if opaque:
        make_opaque(s, seed)
    g = port.random_image_grad(w, h, gseed)
    fr = port.forward(k, s, w, h, BG, threads=0, keep=True)
    st, ref = port.backward(fr["handle"], k, g, s, threads=0)
    port.forward_free(fr["handle"])
    assert st == 0
    sc = scene_f32(s)
    ctx.forward(gpu_kernel_cached(name), **sc, width=w, height=h, background=BG, aux=False)
    got = ctx.backward(gpu_kernel_cached(name), f32(g), n, sc["mu2"], sc["conic"], sc["opacity"], sc["rgb"])
    err = grad_err(got, ref)
    assert err.max() <= GRAD_TOL, f"worst rel err {err.max():.3e} at {np.unravel_index(err.argmax(), err.shape)}"
    strict = rel_err(got, ref, GRAD_FLOOR)
    assert (strict <= GRAD_TOL).mean() >= 0.999
    # the same call with the splat arrays omitted reuses the forward's records
    got2 = ctx.backward(gpu_kernel_cached(name), f32(g), n)
    assert grad_err(got2, ref).max() <= GRAD_TOL
    return err.max()


@pytest.mark.parametrize("name", KERNELS)
@pytest.mark.parametrize("seed", [0, 1])
def test_backward_parity_small(ctx, port, name, seed):
    """All 9 gradients of every splat (the reference checks them against finite differences,
    test_rasterizer.cpp:220-258; here against the oracle's analytic backward)."""
    run_backward_parity(ctx, port, name, 200, 64, 64, seed)


@pytest.mark.parametrize("name", KERNELS + GENERIC)
def test_backward_parity_ragged_dense(ctx, port, name):
    run_backward_parity(ctx, port, name, 3000, 77, 45, 11)


@pytest.mark.parametrize("name", KERNELS + GENERIC[:1])
def test_backward_parity_opaque(ctx, port, name):
    """The alpha clamp blocks the gradient through alpha (rasterizer.cpp:202): clamped and
    unclamped entries mixed in every stream."""
    run_backward_parity(ctx, port, name, 2500, 90, 70, 13, opaque=True)


def test_backward_config1(ctx, port):
    """BASELINE config 1 backward: 10k splats, 256x256, half-cosine-squared."""
    run_backward_parity(ctx, port, "half-cosine-sq", 10000, 256, 256, 0)


@pytest.mark.parametrize("name", ["gaussian", "raised-cosine", "custom:raised-cosine:1.0:0.6:2"])
def test_backward_deterministic_mode_is_bitwise_repeatable(ctx, port, name):
    """The reference's backward is bitwise independent of the thread count because it reduces
    per-tile buffers in a fixed order (rasterizer.cpp:159-165, :219-232; test_rasterizer.cpp:260-273).
    The GPU's float32 reductions arrive in scheduling order; the deterministic mode
    (darbs_cuda_set_deterministic) accumulates them as 64-bit fixed point instead, so two runs are
    bitwise equal — and still the oracle's gradients within the usual tolerance."""
    n, w, h = 6000, 160, 120
    k = oracle_kernel(port, name)
    s = port.random_scene(k, n, w, h, 21)
    g = port.random_image_grad(w, h, 5)
    fr = port.forward(k, s, w, h, BG, threads=0, keep=True)
    st, ref = port.backward(fr["handle"], k, g, s, threads=0)
    port.forward_free(fr["handle"])
    sc = scene_f32(s)
    ctx.set_deterministic(True)
    try:
        runs = []
        for _ in range(3):
            ctx.forward(gpu_kernel_cached(name), **sc, width=w, height=h, background=BG, aux=False)
            runs.append(ctx.backward(gpu_kernel_cached(name), f32(g), n).copy())
    finally:
        ctx.set_deterministic(False)
    assert np.array_equal(runs[0], runs[1]) and np.array_equal(runs[0], runs[2])
    assert grad_err(runs[0], ref).max() <= GRAD_TOL
    # the default mode gives the same sums up to float32 summation order
    ctx.forward(gpu_kernel_cached(name), **sc, width=w, height=h, background=BG, aux=False)
    fast = ctx.backward(gpu_kernel_cached(name), f32(g), n)
    assert grad_err(fast, runs[0].astype(np.float64)).max() <= GRAD_TOL


def test_backward_rejects_mismatched_aux(ctx, port, darbs):
    """contract_violation, test_rasterizer.cpp:176-185."""
    k = port.preset("gaussian")
    s = port.random_scene(k, 10, 32, 32, 2)
    sc = scene_f32(s)
    ctx.forward(gpu_kernel_cached("gaussian"), **sc, width=32, height=32, background=(0, 0, 0), aux=False)
    with pytest.raises(darbs.DarbsError) as e:
        ctx.backward(gpu_kernel_cached("gaussian"), np.zeros((16, 16, 3), np.float32), 10)
    assert e.value.status == 4
    with pytest.raises(darbs.DarbsError) as e:
        ctx.backward(gpu_kernel_cached("gaussian"), np.zeros((32, 32, 3), np.float32), 9)
    assert e.value.status == 4
    # the resident aux belongs to the kernel the forward ran with (include/darbs_cuda.h)
    with pytest.raises(darbs.DarbsError) as e:
        ctx.backward(gpu_kernel_cached("half-cosine-sq"), np.zeros((32, 32, 3), np.float32), 10)
    assert e.value.status == 4


def test_backward_zero_upstream_gives_zero(ctx, port):
    """test_rasterizer.cpp:187-197."""
    k = port.preset("gaussian")
    s = port.random_scene(k, 20, 32, 32, 3)
    ctx.forward(gpu_kernel_cached("gaussian"), **scene_f32(s), width=32, height=32, background=(0, 0, 0), aux=False)
    g = ctx.backward(gpu_kernel_cached("gaussian"), np.zeros((32, 32, 3), np.float32), 20)
    assert np.all(g == 0.0)


def test_backward_is_linear_in_upstream(ctx, port):
    """Size-independent property: backward is linear in dL/dimage."""
    k = port.preset("raised-cosine")
    n, w, h = 2000, 96, 80
    s = port.random_scene(k, n, w, h, 21)
    ctx.forward(gpu_kernel_cached("raised-cosine"), **scene_f32(s), width=w, height=h, background=BG, aux=False)
    g1, g2 = f32(port.random_image_grad(w, h, 1)), f32(port.random_image_grad(w, h, 2))
    a = ctx.backward(gpu_kernel_cached("raised-cosine"), g1, n).astype(np.float64)
    b = ctx.backward(gpu_kernel_cached("raised-cosine"), g2, n).astype(np.float64)
    c = ctx.backward(gpu_kernel_cached("raised-cosine"), f32(2.0 * g1 - 0.5 * g2), n)
    assert rel_err(c, 2.0 * a - 0.5 * b, 1e-3).max() <= 2e-3


def test_work_counters_and_guard_band(ctx, port):
    """Every FP64 re-decision is counted; with the guard band off the FP32 path alone may
    flip a threshold decision, with it on the integer aux matches the oracle."""
    k = port.preset("gaussian")
    n, w, h = 6000, 160, 128
    s = port.random_scene(k, n, w, h, 17)
    ref = port.forward(k, s, w, h, BG, threads=0)
    out = ctx.forward(gpu_kernel_cached("gaussian"), **scene_f32(s), width=w, height=h, background=BG)
    wc = ctx.work_counters()
    assert wc["visits"] == int(ref["processed"].sum())
    assert wc["contributors"] == int(ref["contributors"].sum())
    assert 0 < wc["survivors"] <= wc["entries"] * 8
    assert np.array_equal(out["contributors"], ref["contributors"])
