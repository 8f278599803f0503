"""GPU parity of the loss: darbs_cuda_loss_total against the CPU oracle (src/loss.cpp:173-230).

The device path is FP32 (moments accumulated on values shifted by a per-tile reference), the
reference FP64.  Tolerances, stated once:
  values (total, l1, dssim, mse)     2e-6 absolute
  gradient image                     max |g - g_ref| <= 1e-5 * max |g_ref|  (an absolute bound scaled
                                     to the image's largest gradient: ~100 FP32 ulps of it; measured
                                     3e-6 at 1080p), and the reference's own relative criterion
                                     (tests/test_rasterizer.cpp:242-243)
                                     |g - g_ref| <= 1e-3 * max(|g|, |g_ref|, floor) with
                                     floor = 1e-2 * max |g_ref|
"""
import numpy as np
import pytest

from conftest import f32, rel_err

pytestmark = pytest.mark.gpu

VAL_TOL = 2e-6
GRAD_TOL = 1e-3
GRAD_ABS_TOL = 1e-5


def smooth_pair(w, h, seed, noise=0.02):
    rng = np.random.default_rng(seed)
    yy, xx = np.mgrid[0:h, 0:w]
    img = np.zeros((h, w, 3))
    for _ in range(8):
        cx, cy, s = rng.uniform(0, w), rng.uniform(0, h), rng.uniform(2.0, 0.3 * max(w, h) + 2.0)
        img += np.exp(-((xx - cx) ** 2 + (yy - cy) ** 2) / (2 * s * s))[..., None] * rng.uniform(0, 0.6, 3)
    x = f32(np.clip(img, 0, 1))
    y = f32(np.clip(x + rng.normal(scale=noise, size=x.shape), 0, 1))
    return x, y


def check(ctx, port, x, y, lam, abs_tol=GRAD_ABS_TOL, floor_frac=1e-2, val_tol=VAL_TOL):
    vals, grad = ctx.loss_total(x, y, lam)
    st, ref_vals, ref_grad = port.loss_total(x.astype(np.float64), y.astype(np.float64), lam)
    assert st == 0
    assert np.abs(np.array(vals[:3]) - np.array(ref_vals)).max() <= val_tol, (vals, ref_vals)
    d = x.astype(np.float64) - y
    assert vals[3] == pytest.approx((d * d).mean(), abs=val_tol)
    gmax = max(np.abs(ref_grad).max(), 1e-300)
    abs_err = np.abs(grad - ref_grad).max() / gmax
    # narrower than the window: every tap folds onto a few pixels, var == 0 and the 1/C2-sized
    # terms s_a and d s_d cancel (in the reference too, but at FP64 precision)
    degenerate = min(x.shape[0], x.shape[1]) < 5
    assert abs_err <= (max(1e-4, abs_tol) if degenerate else abs_tol), (x.shape, lam, abs_err)
    err = rel_err(grad, ref_grad, floor_frac * gmax).max()
    assert err <= GRAD_TOL, (x.shape, lam, err)
    return vals, grad


# sizes: below the window (repeated mirror reflection), one tile, ragged tiles, several tiles
SIZES = [(1, 1), (2, 7), (3, 4), (5, 5), (10, 9), (16, 16), (31, 33), (37, 21), (64, 64), (70, 45), (129, 67)]


@pytest.mark.parametrize("size", SIZES, ids=lambda s: f"{s[0]}x{s[1]}")
@pytest.mark.parametrize("lam", [0.0, 0.2, 1.0])
def test_loss_matches_oracle_random_images(ctx, port, size, lam):
    w, h = size
    x, y = f32(port.random_image(w, h, 21)), f32(port.random_image(w, h, 22))
    check(ctx, port, x, y, lam)


@pytest.mark.parametrize("size", [(48, 40), (200, 120)], ids=lambda s: f"{s[0]}x{s[1]}")
def test_loss_matches_oracle_smooth_images(ctx, port, size):
    """Renderer-like images: small local variance, where s_xx - mu^2 cancels."""
    x, y = smooth_pair(*size, seed=3)
    for lam in (0.2, 1.0):
        check(ctx, port, x, y, lam)


def test_loss_known_answers(ctx, port):
    """tests/test_loss.cpp:23-45, :79-86 on the device."""
    x = f32(port.random_image(16, 16, 1))
    for lam in (0.0, 0.2, 1.0):
        vals, grad = ctx.loss_total(x, x, lam)
        assert abs(vals[0]) <= 1e-6 and vals[1] == 0.0 and abs(vals[2]) <= 1e-6
        assert np.abs(grad).max() <= 1e-9
    base = np.minimum(f32(port.random_image(12, 12, 2)), np.float32(0.8))
    vals, _ = ctx.loss_total(base + np.float32(0.1), base, 0.0)
    assert vals[0] == pytest.approx(0.1, abs=1e-6) and vals[1] == pytest.approx(0.1, abs=1e-6)
    x, y = f32(port.random_image(14, 14, 5)), f32(port.random_image(14, 14, 6))
    l0, _ = ctx.loss_total(x, y, 0.0)
    l1, _ = ctx.loss_total(x, y, 1.0)
    mid, _ = ctx.loss_total(x, y, 0.3)
    assert mid[0] == pytest.approx(0.7 * l0[1] + 0.3 * l1[2], abs=1e-6)


def test_loss_values_only_and_errors(ctx, darbs):
    x, y = smooth_pair(40, 30, seed=4)
    with_grad, _ = ctx.loss_total(x, y, 0.2)
    values_only, g = ctx.loss_total(x, y, 0.2, want_grad=False)
    assert g is None and values_only == pytest.approx(with_grad, abs=1e-9)
    with pytest.raises(darbs.DarbsError) as e:
        ctx.loss_total(x, y, 1.5)
    assert e.value.status == 1


def test_loss_full_size_1080p(ctx, port):
    """BASELINE.json's resolution, directly against the oracle (a few seconds of CPU), plus the
    size-independent properties: linear mixing in lambda and device arrays == host arrays."""
    import torch

    w, h = 1920, 1080
    x, y = smooth_pair(w, h, seed=7, noise=0.03)
    vals, grad = check(ctx, port, x, y, 0.2)
    xd, yd = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
    vals_d, grad_d = ctx.loss_total(xd, yd, 0.2)
    assert vals_d == pytest.approx(vals, abs=1e-9)
    assert np.array_equal(grad_d.cpu().numpy(), grad)
    l0, _ = ctx.loss_total(xd, yd, 0.0)
    l1, _ = ctx.loss_total(xd, yd, 1.0)
    assert vals[0] == pytest.approx(0.8 * l0[1] + 0.2 * l1[2], abs=1e-6)
