"""Synthetic 3-D scenes, orbit cameras and learning rates for the training-step workload
(SURVEY.md §8d "input B").  Pure numpy; shared by bench.py and the tests so that the
GPU path and the CPU oracle always consume byte-identical inputs.

The scene is modelled on the reference's proj/data/demo_scene.txt / demo_cameras.txt
scaled up to BASELINE.json's sizes: primitives uniform in a box around the origin,
log-uniform scales that project to a few pixels, orbit cameras at distance 3.132 looking
at the origin with the demo cameras' elevation.
"""
from __future__ import annotations

import numpy as np

ORBIT_DISTANCE = 3.132091953  # |camera centre| of proj/data/demo_cameras.txt
ORBIT_ELEVATION = 0.2873478856  # sin(elevation) of the same cameras


def logit(p):
    return np.log(p / (1.0 - p))


def orbit_camera(view: int, n_views: int, width: int, height: int, focal: float) -> np.ndarray:
    """22 doubles: fx fy cx cy width height + 16 row-major world-to-camera entries
    (include/darbs/scene_io.hpp:16-19).  View v sits at azimuth 2*pi*v/n_views."""
    az = 2.0 * np.pi * view / max(n_views, 1)
    ce = np.sqrt(1.0 - ORBIT_ELEVATION ** 2)
    c = ORBIT_DISTANCE * np.array([ce * np.sin(az), ORBIT_ELEVATION, ce * np.cos(az)])
    f = -c / np.linalg.norm(c)
    r = np.cross([0.0, 1.0, 0.0], f)
    r /= np.linalg.norm(r)
    u = np.cross(f, r)
    rot = np.stack([r, u, f])
    w = np.eye(4)
    w[:3, :3] = rot
    w[:3, 3] = -rot @ c
    return np.concatenate([[focal, focal, width / 2.0, height / 2.0, width, height], w.reshape(-1)])


def scene_b(n: int, seed: int, half_extent=(1.8, 1.0, 1.0), scale_range=(0.002, 0.008)) -> np.ndarray:
    """Ground-truth raw parameters [n, 14] (float32): mu, log scale, quaternion wxyz, logit
    opacity, logit rgb (src/fit3d.cpp:15-25)."""
    rng = np.random.default_rng(seed)
    raw = np.empty((n, 14), dtype=np.float64)
    raw[:, 0:3] = rng.uniform(-1.0, 1.0, (n, 3)) * np.asarray(half_extent)
    raw[:, 3:6] = rng.uniform(np.log(scale_range[0]), np.log(scale_range[1]), (n, 3))
    q = rng.normal(size=(n, 4))
    raw[:, 6:10] = q / np.linalg.norm(q, axis=1, keepdims=True)
    raw[:, 10] = logit(rng.uniform(0.1, 0.95, n))
    raw[:, 11:14] = logit(np.clip(rng.uniform(0.0, 1.0, (n, 3)), 0.01, 0.99))
    return raw.astype(np.float32)


def perturb(raw: np.ndarray, seed: int, amount: float = 0.05, position_scale: float = 0.02) -> np.ndarray:
    """Seeded perturbation of the truth in the spirit of tools/main.cpp:393-407 (positions are
    moved by amount*position_scale so that splats of a few pixels stay near their targets)."""
    rng = np.random.default_rng(seed)
    out = raw.astype(np.float64).copy()
    n = raw.shape[0]
    out[:, 0:3] += amount * position_scale * rng.normal(size=(n, 3))
    out[:, 3:6] += 0.5 * amount * rng.normal(size=(n, 3))
    out[:, 6:10] += 0.5 * amount * rng.normal(size=(n, 4))
    out[:, 10:14] += 2.0 * amount * rng.normal(size=(n, 4))
    return out.astype(np.float32)


def learning_rates(raw: np.ndarray) -> np.ndarray:
    """Per-parameter Adam rates of fit_scene (fit_common.hpp:15-25, fit3d.cpp:54-61,79-84)."""
    mu = raw[:, 0:3].astype(np.float64)
    extent = max(1.0, float(np.linalg.norm(mu.max(axis=0) - mu.min(axis=0))))
    row = np.array([0.00016 * extent] * 3 + [0.005] * 3 + [0.001] * 4 + [0.02] + [0.0025] * 3, dtype=np.float32)
    return np.tile(row, (raw.shape[0], 1))


def sample_workload(n_full: int, width: int, height: int, focal: float, fraction: int):
    """A 1/fraction sample of the full workload at the same splat density and footprint: the
    image shrinks by sqrt(fraction) per side and so does the x/y extent of the box."""
    s = int(round(np.sqrt(fraction)))
    assert s * s == fraction
    return dict(n=n_full // fraction, width=width // s, height=height // s, focal=focal,
                half_extent=(1.8 / s, 1.0 / s, 1.0))


def scene_a(n: int, width: int, height: int, seed: int, cutoff: float = 9.0):
    """The reference's 2-D `random_scene` distribution (benchmarks/bench.cpp:20-46, SURVEY.md 8d
    "input A") with numpy's generator: covariance entries a, c ~ U[0.6, 12] px^2,
    b = U[-0.6, 0.6] sqrt(ac), centres up to 5 px outside the image, depth ~ U[0.5, 9.5], opacity ~
    U[0.1, 0.95], colour ~ U[0, 1]^3; conic and radius as conic_and_radius (geometry.cpp:50-64) gives
    them for a kernel with the given cutoff.  Returns float32 arrays in the forward ABI's layout."""
    rng = np.random.default_rng(seed)
    a = rng.uniform(0.6, 12.0, n)
    c = rng.uniform(0.6, 12.0, n)
    b = rng.uniform(-0.6, 0.6, n) * np.sqrt(a * c)
    det = a * c - b * b
    lam1 = 0.5 * (a + c) + np.sqrt(np.maximum(0.25 * (a - c) ** 2 + b * b, 0.0))
    f32 = lambda x: np.ascontiguousarray(x, dtype=np.float32)  # noqa: E731
    return dict(mu2=f32(np.stack([rng.uniform(-5.0, width + 5.0, n), rng.uniform(-5.0, height + 5.0, n)], axis=1)),
                conic=f32(np.stack([c / det, -b / det, a / det], axis=1)),
                radius=f32(np.ceil(np.sqrt(cutoff) * np.sqrt(lam1))), depth=f32(rng.uniform(0.5, 9.5, n)),
                opacity=f32(rng.uniform(0.1, 0.95, n)), rgb=f32(rng.uniform(0.0, 1.0, (n, 3))))
