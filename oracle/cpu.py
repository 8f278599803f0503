"""ctypes loader for the CPU oracle libraries behind oracle/darbs_cpu.h.

TEST INFRASTRUCTURE, NOT PRODUCT: only tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs may import this module.  The
product package (paper_2501_12369_b200) never does.

``load("port")``      -> oracle/libdarbs_oracle.so   (plain-C restatement)
``load("reference")`` -> oracle/_ref/libdarbs_ref.so (the reference's own sources)
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))

FAMILIES = {
    "gaussian": 0,
    "half-cosine-sq": 1,
    "raised-cosine": 2,
    "mod-sinc": 3,
    "inv-multiquadratic": 4,
}
PRESETS = tuple(FAMILIES)


class Kernel(C.Structure):
    _fields_ = [
        ("family", C.c_int),
        ("beta", C.c_double),
        ("xi", C.c_double),
        ("lobes", C.c_int),
        ("cutoff", C.c_double),
        ("unbounded", C.c_int),
    ]


_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int32)
_lp = C.POINTER(C.c_int64)


def _d(a):
    return None if a is None else a.ctypes.data_as(_dp)


def _i(a):
    return None if a is None else a.ctypes.data_as(_ip)


def _l(a):
    return None if a is None else a.ctypes.data_as(_lp)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


class Scene:
    """Projected 2-D splats in the reference's FP64 element type (SoA)."""

    def __init__(self, mu2, cov2, conic, radius, depth, opacity, rgb):
        self.mu2, self.cov2, self.conic = _f64(mu2), (None if cov2 is None else _f64(cov2)), _f64(conic)
        self.radius, self.depth = _f64(radius), _f64(depth)
        self.opacity, self.rgb = _f64(opacity), _f64(rgb)

    @property
    def n(self):
        return int(self.depth.shape[0])

    def take(self, idx):
        return Scene(self.mu2[idx], None if self.cov2 is None else self.cov2[idx], self.conic[idx],
                     self.radius[idx], self.depth[idx], self.opacity[idx], self.rgb[idx])


class Oracle:
    def __init__(self, path):
        self.path = path
        lib = C.CDLL(path)
        self.lib = lib
        lib.darbs_cpu_kind.restype = C.c_char_p
        lib.darbs_cpu_default_psi.restype = C.c_double
        lib.darbs_cpu_default_psi.argtypes = [C.c_char_p]
        lib.darbs_cpu_make_kernel.argtypes = [C.c_int, C.c_double, C.c_double, C.c_int, C.POINTER(Kernel)]
        lib.darbs_cpu_kernel_preset.argtypes = [C.c_char_p, C.POINTER(Kernel)]
        lib.darbs_cpu_eval.argtypes = [C.POINTER(Kernel), C.c_int, _dp, _dp, _dp]
        lib.darbs_cpu_conic_and_radius.argtypes = [C.POINTER(Kernel), C.c_int, _dp, _dp, _dp, _dp]
        lib.darbs_cpu_random_scene.argtypes = [C.POINTER(Kernel), C.c_int, C.c_int, C.c_int, C.c_uint64,
                                               C.c_int, _dp, _dp, _dp, _dp, _dp, _dp, _dp]
        lib.darbs_cpu_random_image_grad.argtypes = [C.c_int, C.c_int, C.c_uint64, C.c_int, _dp]
        lib.darbs_cpu_random_image_grad.restype = None
        lib.darbs_cpu_bin.restype = C.c_int64
        lib.darbs_cpu_bin.argtypes = [C.c_int, _dp, _dp, _dp, _dp, C.c_int, C.c_int, _lp, _ip, C.c_int64, _ip]
        lib.darbs_cpu_forward.restype = C.c_void_p
        lib.darbs_cpu_forward.argtypes = [C.POINTER(Kernel), C.c_int, _dp, _dp, _dp, _dp, _dp, _dp, C.c_int,
                                          C.c_int, _dp, C.c_int, _dp, _dp, _ip, _ip, _ip]
        lib.darbs_cpu_forward_free.argtypes = [C.c_void_p]
        lib.darbs_cpu_forward_free.restype = None
        lib.darbs_cpu_oracle_forward.argtypes = [C.POINTER(Kernel), C.c_int, _dp, _dp, _dp, _dp, _dp, _dp,
                                                 C.c_int, C.c_int, _dp, _dp]
        lib.darbs_cpu_backward.argtypes = [C.c_void_p, C.POINTER(Kernel), C.c_int, C.c_int, _dp, C.c_int,
                                           _dp, _dp, _dp, _dp, C.c_int, _dp]
        lib.darbs_cpu_realize.argtypes = [C.c_int, _dp, _dp]
        lib.darbs_cpu_realize.restype = None
        lib.darbs_cpu_project.argtypes = [C.POINTER(Kernel), C.c_double, C.c_double, C.c_int, _dp, _dp, _ip,
                                          _dp, _dp, _dp, _dp, _dp]
        lib.darbs_cpu_backward_projection.argtypes = [C.c_double, C.c_int, _dp, _dp, _dp, _dp, _dp, _dp, _dp]
        lib.darbs_cpu_backward_projection.restype = None
        lib.darbs_cpu_param_grads.argtypes = [C.c_double, C.c_int, _ip, _dp, _dp, _dp, _dp, _dp, _dp, _dp]
        lib.darbs_cpu_param_grads.restype = None
        lib.darbs_cpu_adam_step.argtypes = [C.c_int64, _dp, _dp, _dp, _dp, _dp, C.c_int]
        lib.darbs_cpu_loss_total.argtypes = [C.c_int, C.c_int, _dp, _dp, C.c_double, _dp, _dp]
        lib.darbs_cpu_ssim.argtypes = [C.c_int, C.c_int, _dp, _dp, _dp]
        lib.darbs_cpu_random_image.argtypes = [C.c_int, C.c_int, C.c_uint64, C.c_int, _dp]
        lib.darbs_cpu_random_image.restype = None
        if hasattr(lib, "darbs_cpu_write_scene"):  # file formats: reference build only
            lib.darbs_cpu_write_scene.argtypes = [C.c_char_p, C.c_int, _dp]
            lib.darbs_cpu_read_scene.argtypes = [C.c_char_p, C.c_int, _dp]
            lib.darbs_cpu_write_cameras.argtypes = [C.c_char_p, C.c_int, _dp]
            lib.darbs_cpu_write_image.argtypes = [C.c_char_p, C.c_int, C.c_int, _dp, C.c_int]
        if hasattr(lib, "darbs_cpu_fit_scene"):  # the callers of the hot path: reference build only
            lib.darbs_cpu_render_scene.argtypes = [C.POINTER(Kernel), C.c_double, C.c_int, _dp, _dp, _dp, C.c_int, _dp]
            lib.darbs_cpu_fit_scene.argtypes = [C.POINTER(Kernel), C.c_double, C.c_int, _dp, C.c_int, _dp, _dp, _dp,
                                                _dp, _dp, _dp, _dp]
            lib.darbs_cpu_fit_image.argtypes = [C.POINTER(Kernel), C.c_int, C.c_int, _dp, C.c_int, _dp, _dp, _dp,
                                                _dp, _dp]
            lib.darbs_cpu_read_cameras.argtypes = [C.c_char_p, C.c_int, _dp]

    # ------------------------------------------------------------------ kernel
    @property
    def kind(self):
        return self.lib.darbs_cpu_kind().decode()

    def make_kernel(self, family, beta, xi, lobes=1):
        k = Kernel()
        fam = FAMILIES[family] if isinstance(family, str) else int(family)
        st = self.lib.darbs_cpu_make_kernel(fam, beta, xi, lobes, C.byref(k))
        return st, k

    def preset(self, name):
        k = Kernel()
        st = self.lib.darbs_cpu_kernel_preset(name.encode(), C.byref(k))
        if st != 0:
            raise KeyError(name)
        return k

    def default_psi(self, name):
        return float(self.lib.darbs_cpu_default_psi(name.encode()))

    def eval(self, k, dm2):
        dm2 = _f64(np.atleast_1d(dm2))
        w = np.empty_like(dm2)
        dw = np.empty_like(dm2)
        st = self.lib.darbs_cpu_eval(C.byref(k), dm2.size, _d(dm2), _d(w), _d(dw))
        return st, w, dw

    def conic_and_radius(self, k, cov2):
        cov2 = _f64(cov2).reshape(-1, 3)
        n = cov2.shape[0]
        conic = np.full((n, 3), np.nan)
        radius = np.full(n, np.nan)
        lam = np.full((n, 2), np.nan)
        st = self.lib.darbs_cpu_conic_and_radius(C.byref(k), n, _d(cov2), _d(conic), _d(radius), _d(lam))
        return st, conic, radius, lam

    # ---------------------------------------------------------------- fixtures
    def random_scene(self, k, count, width, height, seed, round_f32=True):
        mu2 = np.empty((count, 2))
        cov2 = np.empty((count, 3))
        conic = np.empty((count, 3))
        radius = np.empty(count)
        depth = np.empty(count)
        opacity = np.empty(count)
        rgb = np.empty((count, 3))
        st = self.lib.darbs_cpu_random_scene(C.byref(k), count, width, height, seed, int(round_f32), _d(mu2),
                                             _d(cov2), _d(conic), _d(radius), _d(depth), _d(opacity), _d(rgb))
        if st != 0:
            raise RuntimeError(f"random_scene status {st}")
        return Scene(mu2, cov2, conic, radius, depth, opacity, rgb)

    def random_image_grad(self, width, height, seed, round_f32=True):
        g = np.empty((height, width, 3))
        self.lib.darbs_cpu_random_image_grad(width, height, seed, int(round_f32), _d(g))
        return g

    # -------------------------------------------------------------- rasterizer
    def bin(self, s: Scene, width, height):
        tiles = ((width + 15) // 16) * ((height + 15) // 16)
        offsets = np.zeros(tiles + 1, dtype=np.int64)
        order = np.zeros(max(s.n, 1), dtype=np.int32)
        k = self.lib.darbs_cpu_bin(s.n, _d(s.mu2), _d(s.conic), _d(s.radius), _d(s.depth), width, height,
                                   _l(offsets), None, 0, _i(order))
        plist = np.zeros(max(int(k), 1), dtype=np.int32)
        k2 = self.lib.darbs_cpu_bin(s.n, _d(s.mu2), _d(s.conic), _d(s.radius), _d(s.depth), width, height,
                                    _l(offsets), _i(plist), int(k), _i(order))
        assert k2 == k
        return offsets, plist[: int(k)], order[: s.n]

    def forward(self, k, s: Scene, width, height, background, threads=1, keep=False):
        px = width * height
        image = np.empty((height, width, 3))
        t_final = np.empty((height, width))
        processed = np.empty((height, width), dtype=np.int32)
        contributors = np.empty((height, width), dtype=np.int32)
        skipped = C.c_int32(0)
        bg = _f64(background)
        h = self.lib.darbs_cpu_forward(C.byref(k), s.n, _d(s.mu2), _d(s.conic), _d(s.radius), _d(s.depth),
                                       _d(s.opacity), _d(s.rgb), width, height, _d(bg), threads, _d(image),
                                       _d(t_final), _i(processed), _i(contributors), C.byref(skipped))
        if not h:
            raise RuntimeError("oracle forward failed")
        out = dict(image=image, t_final=t_final, processed=processed, contributors=contributors,
                   skipped=int(skipped.value), px=px)
        if keep:
            out["handle"] = h
        else:
            self.lib.darbs_cpu_forward_free(h)
        return out

    def forward_free(self, handle):
        self.lib.darbs_cpu_forward_free(handle)

    def oracle_forward(self, k, s: Scene, width, height, background):
        image = np.empty((height, width, 3))
        bg = _f64(background)
        st = self.lib.darbs_cpu_oracle_forward(C.byref(k), s.n, _d(s.mu2), _d(s.conic), _d(s.radius),
                                               _d(s.depth), _d(s.opacity), _d(s.rgb), width, height, _d(bg),
                                               _d(image))
        assert st == 0
        return image

    def backward(self, handle, k, grad_image, s: Scene, threads=1, n=None):
        g = _f64(grad_image)
        gh, gw = g.shape[0], g.shape[1]
        n = s.n if n is None else n
        grads = np.zeros((max(n, 1), 9))
        st = self.lib.darbs_cpu_backward(handle, C.byref(k), gw, gh, _d(g), n, _d(s.mu2), _d(s.conic),
                                         _d(s.opacity), _d(s.rgb), threads, _d(grads))
        return st, grads[:n]

    # ---------------------------------------------------------------- geometry
    def realize(self, raw):
        raw = _f64(raw).reshape(-1, 14)
        prims = np.empty_like(raw)
        self.lib.darbs_cpu_realize(raw.shape[0], _d(raw), _d(prims))
        return prims

    def project(self, k, psi, prims, camera, dilation=0.3):
        prims = _f64(prims).reshape(-1, 14)
        cam = _f64(camera).reshape(22)
        n = prims.shape[0]
        valid = np.zeros(n, dtype=np.int32)
        mu2 = np.zeros((n, 2))
        cov2 = np.zeros((n, 3))
        conic = np.zeros((n, 3))
        radius = np.zeros(n)
        depth = np.zeros(n)
        st = self.lib.darbs_cpu_project(C.byref(k), psi, dilation, n, _d(prims), _d(cam), _i(valid), _d(mu2),
                                        _d(cov2), _d(conic), _d(radius), _d(depth))
        return st, dict(valid=valid, mu2=mu2, cov2=cov2, conic=conic, radius=radius, depth=depth)

    def backward_projection(self, psi, grad_cov2, grad_mu2, prims, camera):
        prims = _f64(prims).reshape(-1, 14)
        n = prims.shape[0]
        gc = _f64(grad_cov2).reshape(n, 4)
        gm = _f64(grad_mu2).reshape(n, 2)
        cam = _f64(camera).reshape(22)
        d_mu = np.zeros((n, 3))
        d_scale = np.zeros((n, 3))
        d_rot = np.zeros((n, 4))
        self.lib.darbs_cpu_backward_projection(psi, n, _d(gc), _d(gm), _d(prims), _d(cam), _d(d_mu),
                                               _d(d_scale), _d(d_rot))
        return d_mu, d_scale, d_rot

    def param_grads(self, psi, owner, splat_grads, conic, opacity, rgb, prims, camera, out=None):
        prims = _f64(prims).reshape(-1, 14)
        owner = np.ascontiguousarray(owner, dtype=np.int32)
        sg = _f64(splat_grads).reshape(-1, 9)
        conic, opacity, rgb = _f64(conic), _f64(opacity), _f64(rgb)
        cam = _f64(camera).reshape(22)
        if out is None:
            out = np.zeros_like(prims)
        self.lib.darbs_cpu_param_grads(psi, owner.size, _i(owner), _d(sg), _d(conic), _d(opacity), _d(rgb),
                                       _d(prims), _d(cam), _d(out))
        return out

    def random_image(self, width, height, seed, round_f32=True):
        """tests/test_loss.cpp:13-19: U[0,1) per value from mt19937_64(seed); (h, w, 3)."""
        img = np.empty((height, width, 3))
        self.lib.darbs_cpu_random_image(width, height, seed, int(round_f32), _d(img))
        return img

    def loss_total(self, rendered, target, lam, want_grad=True):
        """loss.cpp:173-230 -> (status, (total, l1, dssim), grad or None); images are (h, w, 3)."""
        rendered, target = _f64(rendered), _f64(target)
        h, w = rendered.shape[:2]
        out = np.zeros(3)
        grad = np.empty_like(rendered) if want_grad else None
        st = self.lib.darbs_cpu_loss_total(w, h, _d(rendered), _d(target), float(lam), _d(out),
                                           _d(grad) if want_grad else None)
        return st, tuple(out), grad

    def ssim(self, a, b):
        a, b = _f64(a), _f64(b)
        h, w = a.shape[:2]
        out = np.zeros(1)
        st = self.lib.darbs_cpu_ssim(w, h, _d(a), _d(b), _d(out))
        return st, float(out[0])

    # ---- file formats (reference build only)
    def write_scene(self, path, prims):
        prims = _f64(prims)
        return self.lib.darbs_cpu_write_scene(os.fsencode(path), prims.shape[0], _d(prims))

    def read_scene(self, path, capacity=4096):
        out = np.zeros((capacity, 14))
        n = self.lib.darbs_cpu_read_scene(os.fsencode(path), capacity, _d(out))
        return n, out[:max(n, 0)]

    def write_cameras(self, path, cams22):
        cams22 = _f64(cams22).reshape(-1, 22)
        return self.lib.darbs_cpu_write_cameras(os.fsencode(path), cams22.shape[0], _d(cams22))

    def write_image(self, path, img, ppm=False):
        img = _f64(img)
        return self.lib.darbs_cpu_write_image(os.fsencode(path), img.shape[1], img.shape[0], _d(img), int(ppm))

    # ---- the reference's callers of the hot path (reference build only)
    @staticmethod
    def fit_config(lam=0.2, lr_position=0.00016, lr_scale=0.005, lr_rotation=0.001, lr_opacity=0.02,
                   lr_color=0.0025, iters=100, seed=1, threads=1):
        """FitConfig, include/darbs/fit_common.hpp:15-25 (its defaults)."""
        return np.array([lam, lr_position, lr_scale, lr_rotation, lr_opacity, lr_color, iters, seed, threads],
                        dtype=np.float64)

    def read_cameras(self, path, capacity=64):
        out = np.zeros((capacity, 22))
        n = self.lib.darbs_cpu_read_cameras(os.fsencode(path), capacity, _d(out))
        return n, out[:max(n, 0)]

    def render_scene(self, k, psi, prims, camera, background=(0.0, 0.0, 0.0), threads=1):
        """render_scene, fit3d.cpp:29-40 -> (status, image (h, w, 3))."""
        prims, camera = _f64(prims), _f64(camera)
        img = np.zeros((int(camera[5]), int(camera[4]), 3))
        bg = np.asarray(background, dtype=np.float64)
        st = self.lib.darbs_cpu_render_scene(C.byref(k), float(psi), prims.shape[0], _d(prims), _d(camera), _d(bg),
                                             threads, _d(img))
        return st, img

    def fit_scene(self, k, psi, init_prims, cameras22, targets, cfg):
        """fit_scene, fit3d.cpp:42-203.  targets: list of (h, w, 3) images, one per camera."""
        init_prims, cameras22 = _f64(init_prims), _f64(cameras22).reshape(-1, 22)
        n, nv, iters = init_prims.shape[0], cameras22.shape[0], max(int(cfg[6]), 1)
        tg = np.concatenate([_f64(t).reshape(-1) for t in targets])
        curves, finals = np.zeros((4, iters)), np.zeros(3)
        pv, out = np.zeros(nv), np.zeros((n, 14))
        st = self.lib.darbs_cpu_fit_scene(C.byref(k), float(psi), n, _d(init_prims), nv, _d(cameras22), _d(tg),
                                          _d(_f64(cfg)), _d(curves), _d(finals), _d(pv), _d(out))
        return st, dict(loss=curves[0], l1=curves[1], dssim=curves[2], psnr=curves[3], final_mse=finals[0],
                        final_psnr=finals[1], final_ssim=finals[2], per_view_psnr=pv, primitives=out)

    def fit_image(self, k, target, n_splats, cfg):
        """fit_image, fit2d.cpp:45-188."""
        target = _f64(target)
        h, w = target.shape[:2]
        iters = max(int(cfg[6]), 1)
        curves, finals = np.zeros((4, iters)), np.zeros(3)
        rendered, splats = np.zeros_like(target), np.zeros((n_splats, 9))
        st = self.lib.darbs_cpu_fit_image(C.byref(k), w, h, _d(target), n_splats, _d(_f64(cfg)), _d(curves),
                                          _d(finals), _d(rendered), _d(splats))
        return st, dict(loss=curves[0], l1=curves[1], dssim=curves[2], psnr=curves[3], final_mse=finals[0],
                        final_psnr=finals[1], final_ssim=finals[2], rendered=rendered, splats=splats)

    def adam_step(self, params, grads, m, v, lrs, t):
        params, grads, m, v, lrs = (_f64(a).copy() for a in (params, grads, m, v, lrs))
        st = self.lib.darbs_cpu_adam_step(params.size, _d(params), _d(grads), _d(m), _d(v), _d(lrs), t)
        return st, params, m, v


_PATHS = {
    "port": os.path.join(_HERE, "libdarbs_oracle.so"),
    "reference": os.path.join(_HERE, "_ref", "libdarbs_ref.so"),
}
_CACHE: dict = {}


def build(ref: bool = True) -> None:
    """Compile the checkers (gcc/g++ via oracle/Makefile).  Building is not using."""
    subprocess.run(["make", "-C", _HERE, "port"], check=True, capture_output=True)
    if ref:
        subprocess.run(["make", "-C", _HERE, "ref"], check=True, capture_output=True)


def available(kind: str) -> bool:
    return os.path.exists(_PATHS[kind])


def load(kind: str = "port") -> Oracle:
    if kind not in _CACHE:
        if kind == "port" and not available("port"):
            build(ref=False)
        if not available(kind):
            raise FileNotFoundError(_PATHS[kind])
        _CACHE[kind] = Oracle(_PATHS[kind])
    return _CACHE[kind]
