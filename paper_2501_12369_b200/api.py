"""ctypes binding of include/darbs_cuda.h.

Arrays may be numpy arrays (``DARBS_HOST``: the library stages them) or torch
CUDA tensors (``DARBS_DEVICE``: zero-copy, asynchronous on the context's
stream).  All arrays of one call must live in the same space.  Every non-OK
status raises :class:`DarbsError` carrying the status code, so tests can assert
the reference's error taxonomy (``include/darbs/errors.hpp``).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HOST, DEVICE = 0, 1

OK, INVALID_PARAMETER, NUMERIC_ERROR, IO_ERROR, CONTRACT_VIOLATION, CUDA_ERROR = range(6)
_STATUS_NAMES = {
    OK: "ok",
    INVALID_PARAMETER: "invalid_parameter",
    NUMERIC_ERROR: "numeric_error",
    IO_ERROR: "io_error",
    CONTRACT_VIOLATION: "contract_violation",
    CUDA_ERROR: "cuda_error",
}

FAMILIES = {
    "gaussian": 0,
    "half-cosine": 1,
    "raised-cosine": 2,
    "mod-sinc": 3,
    "inv-multiquadratic": 4,
}
PRESETS = ("gaussian", "half-cosine-sq", "raised-cosine", "mod-sinc", "inv-multiquadratic")

_HERE = os.path.dirname(os.path.abspath(__file__))


def lib_path() -> str:
    return os.path.join(_HERE, "libdarbs_cuda.so")


class DarbsError(RuntimeError):
    def __init__(self, status: int, message: str):
        super().__init__(f"{_STATUS_NAMES.get(status, status)}: {message}")
        self.status = status
        self.message = message


class KernelSpec(C.Structure):
    """darbs_kernel_spec == KernelSpec of include/darbs/kernel.hpp:20-33."""

    _fields_ = [
        ("family", C.c_int32),
        ("beta", C.c_double),
        ("xi", C.c_double),
        ("lobes", C.c_int32),
        ("cutoff", C.c_double),
        ("unbounded", C.c_int32),
    ]


def _load():
    path = lib_path()
    if not os.path.exists(path):
        raise ImportError(
            f"{path} is missing: build it with `make -C paper_2501_12369_b200/csrc` "
            "(or __graft_entry__.build()). There is no CPU fallback."
        )
    lib = C.CDLL(path)
    vp, i32, i64, dbl = C.c_void_p, C.c_int, C.c_int64, C.c_double
    ks = C.POINTER(KernelSpec)
    lib.darbs_cuda_version.restype = C.c_char_p
    lib.darbs_cuda_create.argtypes = [i32, C.POINTER(vp)]
    lib.darbs_cuda_destroy.argtypes = [vp]
    lib.darbs_cuda_destroy.restype = None
    lib.darbs_cuda_last_error.argtypes = [vp]
    lib.darbs_cuda_last_error.restype = C.c_char_p
    lib.darbs_cuda_set_stream.argtypes = [vp, vp]
    lib.darbs_cuda_synchronize.argtypes = [vp]
    lib.darbs_cuda_launch_count.argtypes = [vp]
    lib.darbs_cuda_launch_count.restype = i64
    lib.darbs_cuda_set_exact_decisions.argtypes = [vp, i32]
    lib.darbs_cuda_set_deterministic.argtypes = [vp, i32]
    lib.darbs_cuda_set_cull_segment.argtypes = [vp, i32]
    lib.darbs_cuda_set_entry_capacity.argtypes = [vp, i64]
    lib.darbs_cuda_make_kernel.argtypes = [i32, dbl, dbl, i32, ks]
    lib.darbs_cuda_kernel_preset.argtypes = [C.c_char_p, ks]
    lib.darbs_cuda_default_psi.argtypes = [C.c_char_p]
    lib.darbs_cuda_default_psi.restype = dbl
    lib.darbs_cuda_eval.argtypes = [vp, ks, i64, vp, vp, vp, i32, i32]
    lib.darbs_cuda_bin.argtypes = [vp, i64, vp, vp, vp, vp, i32, i32, C.POINTER(i64), vp, vp, vp, vp, i64, i32]
    lib.darbs_cuda_forward.argtypes = [vp, ks, i64, vp, vp, vp, vp, vp, vp, i32, i32, C.POINTER(C.c_float),
                                       vp, vp, vp, vp, C.POINTER(C.c_int32), i32]
    lib.darbs_cuda_backward.argtypes = [vp, ks, i32, i32, vp, i64, vp, vp, vp, vp, vp, i32]
    lib.darbs_cuda_realize.argtypes = [vp, i64, vp, vp, i32]
    lib.darbs_cuda_project.argtypes = [vp, ks, dbl, dbl, i64, vp, C.POINTER(dbl), vp, vp, vp, vp, vp, vp, i32]
    lib.darbs_cuda_backward_projection.argtypes = [vp, dbl, i64, vp, vp, vp, C.POINTER(dbl), vp, vp, vp, i32]
    lib.darbs_cuda_evaluate_view.argtypes = [vp, ks, dbl, i64, vp, C.POINTER(dbl), C.POINTER(C.c_float), vp,
                                             dbl, vp, vp, vp, C.POINTER(dbl), i32, i32]
    lib.darbs_cuda_pop_loss.argtypes = [vp, C.POINTER(dbl)]
    lib.darbs_cuda_prefetch_target.argtypes = [vp, vp, i64]
    lib.darbs_cuda_microbench.argtypes = [vp, C.POINTER(dbl)]
    lib.darbs_cuda_adam_step.argtypes = [vp, i64, vp, vp, vp, vp, vp, i32, i32]
    lib.darbs_cuda_loss_total.argtypes = [vp, i32, i32, vp, vp, dbl, C.POINTER(dbl), vp, i32]
    lib.darbs_cuda_device_alloc.argtypes = [vp, C.c_uint64, C.POINTER(vp)]
    lib.darbs_cuda_device_free.argtypes = [vp, vp]
    lib.darbs_cuda_upload.argtypes = [vp, vp, vp, C.c_uint64]
    lib.darbs_cuda_download.argtypes = [vp, vp, vp, C.c_uint64]
    lib.darbs_cuda_device_zero.argtypes = [vp, vp, C.c_uint64]
    lib.darbs_cuda_set_accumulate.argtypes = [vp, i32]
    lib.darbs_cuda_comm_unique_id.argtypes = [C.c_char_p]
    lib.darbs_cuda_comm_init.argtypes = [vp, C.c_char_p, i32, i32]
    lib.darbs_cuda_comm_destroy.argtypes = [vp]
    lib.darbs_cuda_allreduce_adam_step.argtypes = [vp, i64, vp, vp, vp, vp, vp, i32]
    lib.darbs_cuda_train_step.argtypes = [vp, C.POINTER(KernelSpec), dbl, i64, vp, vp, vp, vp, vp, i32, C.POINTER(dbl),
                                          C.POINTER(vp), dbl, C.POINTER(C.c_float), i32, i32, C.POINTER(dbl)]
    lib.darbs_cuda_set_stage_timing.argtypes = [vp, i32]
    lib.darbs_cuda_stage_times.argtypes = [vp, C.POINTER(dbl)]
    lib.darbs_cuda_work_counters.argtypes = [vp, C.POINTER(i64)]
    return lib


_lib = _load()

EXPORTED_SYMBOLS = (
    "darbs_cuda_version darbs_cuda_create darbs_cuda_destroy darbs_cuda_last_error darbs_cuda_set_stream "
    "darbs_cuda_synchronize darbs_cuda_launch_count darbs_cuda_set_exact_decisions darbs_cuda_set_deterministic darbs_cuda_set_cull_segment darbs_cuda_set_entry_capacity darbs_cuda_make_kernel "
    "darbs_cuda_kernel_preset darbs_cuda_default_psi darbs_cuda_eval darbs_cuda_bin darbs_cuda_forward "
    "darbs_cuda_backward darbs_cuda_realize darbs_cuda_project darbs_cuda_backward_projection "
    "darbs_cuda_evaluate_view darbs_cuda_prefetch_target darbs_cuda_pop_loss darbs_cuda_adam_step darbs_cuda_set_stage_timing darbs_cuda_stage_times "
    "darbs_cuda_work_counters darbs_cuda_microbench darbs_cuda_loss_total darbs_cuda_device_alloc "
    "darbs_cuda_device_free darbs_cuda_upload darbs_cuda_download darbs_cuda_device_zero darbs_cuda_set_accumulate "
    "darbs_cuda_comm_unique_id darbs_cuda_comm_init darbs_cuda_comm_destroy darbs_cuda_train_step "
    "darbs_cuda_allreduce_adam_step"
).split()


def version() -> str:
    return _lib.darbs_cuda_version().decode()


def _raise(status: int, ctx=None):
    msg = _lib.darbs_cuda_last_error(ctx).decode()
    raise DarbsError(status, msg)


def comm_unique_id() -> bytes:
    """ncclGetUniqueId: rank 0 makes it and hands it to the other ranks (darbs_cuda_comm_unique_id)."""
    buf = C.create_string_buffer(128)
    st = _lib.darbs_cuda_comm_unique_id(buf)
    if st != 0:
        _raise(st)
    return buf.raw


def make_kernel(family, beta: float, xi: float, lobes: int = 1) -> KernelSpec:
    """make_kernel, src/kernel.cpp:42-65."""
    fam = FAMILIES[family] if isinstance(family, str) else int(family)
    k = KernelSpec()
    st = _lib.darbs_cuda_make_kernel(fam, beta, xi, lobes, C.byref(k))
    if st != OK:
        _raise(st)
    return k


def kernel_preset(name: str) -> KernelSpec:
    """kernel_preset, src/kernel.cpp:223-240."""
    k = KernelSpec()
    st = _lib.darbs_cuda_kernel_preset(name.encode(), C.byref(k))
    if st != OK:
        _raise(st)
    return k


def default_psi(name: str) -> float:
    return float(_lib.darbs_cuda_default_psi(name.encode()))


def _is_torch(a) -> bool:
    return a is not None and type(a).__module__.startswith("torch")


class _Args:
    """Collects the arrays of one call, checks they share a memory space."""

    def __init__(self):
        self.space = None
        self.keep = []

    def _note(self, space):
        if self.space is None:
            self.space = space
        elif self.space != space:
            raise TypeError("all arrays of one call must be numpy (host) or torch CUDA (device), not a mix")

    def ptr(self, a, dtype, count=None):
        if a is None:
            return None
        if _is_torch(a):
            import torch

            want = {np.float32: torch.float32, np.int32: torch.int32, np.uint64: torch.int64,
                    np.int64: torch.int64}[dtype]
            if not a.is_cuda:
                raise TypeError("torch tensors must live on the GPU (pass numpy arrays for host data)")
            if a.dtype != want or not a.is_contiguous():
                raise TypeError(f"expected contiguous {want} tensor, got {a.dtype}")
            if count is not None and a.numel() != count:
                raise ValueError(f"expected {count} elements, got {a.numel()}")
            self._note(DEVICE)
            self.keep.append(a)
            return C.c_void_p(a.data_ptr())
        arr = np.ascontiguousarray(a, dtype=dtype)
        if count is not None and arr.size != count:
            raise ValueError(f"expected {count} elements, got {arr.size}")
        self._note(HOST)
        self.keep.append(arr)
        return C.c_void_p(arr.ctypes.data)

    def inout(self, a, dtype, count=None):
        """Pointer to an array the call updates in place: no silent copies."""
        if a is not None and not _is_torch(a):
            if not (isinstance(a, np.ndarray) and a.dtype == dtype and a.flags.c_contiguous and a.flags.writeable):
                raise TypeError(f"in/out arrays must be writable contiguous {np.dtype(dtype)} numpy arrays")
        return self.ptr(a, dtype, count)

    def out(self, like, shape, dtype):
        """Allocate an output in the same space as ``like``."""
        if _is_torch(like):
            import torch

            tdt = {np.float32: torch.float32, np.int32: torch.int32, np.uint64: torch.int64}[dtype]
            t = torch.empty(shape, dtype=tdt, device=like.device)
            self._note(DEVICE)
            self.keep.append(t)
            return t, C.c_void_p(t.data_ptr())
        arr = np.empty(shape, dtype=dtype)
        self._note(HOST)
        self.keep.append(arr)
        return arr, C.c_void_p(arr.ctypes.data)


def _cam(camera):
    cam = np.ascontiguousarray(camera, dtype=np.float64).reshape(22)
    return cam, cam.ctypes.data_as(C.POINTER(C.c_double))


class Context:
    """One darbs_cuda_ctx: a GPU, a stream and the grow-only device workspace."""

    def __init__(self, device: int = 0):
        h = C.c_void_p()
        st = _lib.darbs_cuda_create(int(device), C.byref(h))
        if st != OK:
            _raise(st)
        self._h = h
        self.device = int(device)

    def close(self):
        if getattr(self, "_h", None):
            _lib.darbs_cuda_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def _check(self, st):
        if st != OK:
            _raise(st, self._h)

    # ------------------------------------------------------------ plumbing
    def set_stream(self, cuda_stream: int | None):
        self._check(_lib.darbs_cuda_set_stream(self._h, C.c_void_p(cuda_stream or 0)))

    def use_torch_stream(self):
        """Run on torch's current stream.  torch's default stream is the legacy NULL stream,
        which the ABI spells cudaStreamLegacy (1) because NULL means "the context's own"."""
        import torch

        h = torch.cuda.current_stream(self.device).cuda_stream
        self.set_stream(h if h else 1)

    def synchronize(self):
        self._check(_lib.darbs_cuda_synchronize(self._h))

    def launch_count(self) -> int:
        return int(_lib.darbs_cuda_launch_count(self._h))

    def set_exact_decisions(self, enabled: bool):
        self._check(_lib.darbs_cuda_set_exact_decisions(self._h, int(bool(enabled))))

    def set_deterministic(self, enabled: bool):
        """Order-independent fixed-point accumulation of gradients and loss sums (bitwise repeatable)."""
        self._check(_lib.darbs_cuda_set_deterministic(self._h, int(bool(enabled))))

    def set_entry_capacity(self, entries: int):
        """Promise K <= entries for the following evaluate_view / train_step calls: they stop waiting for K
        (0 restores the wait).  A view that breaks the promise raises contract_violation when its loss is collected."""
        self._check(_lib.darbs_cuda_set_entry_capacity(self._h, int(entries)))

    def set_cull_segment(self, entries: int):
        """List entries per tile the cull kernel covers before the forward extends streams by itself (0: default)."""
        self._check(_lib.darbs_cuda_set_cull_segment(self._h, int(entries)))

    def set_stage_timing(self, enabled: bool):
        self._check(_lib.darbs_cuda_set_stage_timing(self._h, int(bool(enabled))))

    def stage_times(self) -> dict:
        out = (C.c_double * 8)()
        self._check(_lib.darbs_cuda_stage_times(self._h, out))
        names = ["preprocess", "binning", "render_fwd", "loss", "render_bwd", "preprocess_bwd", "adam", "cull"]
        return {k: float(out[i]) for i, k in enumerate(names)}

    def microbench(self) -> dict:
        out = (C.c_double * 8)()
        self._check(_lib.darbs_cuda_microbench(self._h, out))
        return dict(ffma_per_s=float(out[0]), mufu_per_s=float(out[1]), sm_mhz=float(out[2]), sms=int(out[3]),
                    ffma_imm_per_s=float(out[4]), ffma2_per_s=float(out[5]))

    def work_counters(self) -> dict:
        out = (C.c_int64 * 8)()
        self._check(_lib.darbs_cuda_work_counters(self._h, out))
        names = ["entries", "visits", "contributors", "survivors", "exact", "tfloor", "composited"]
        return {k: int(out[i]) for i, k in enumerate(names)}

    # -------------------------------------------------------------- kernel
    def eval(self, kernel: KernelSpec, dm2, exact: bool = False):
        a = _Args()
        n = dm2.numel() if _is_torch(dm2) else np.asarray(dm2).size
        p = a.ptr(dm2, np.float32)
        w, pw = a.out(dm2, (n,), np.float32)
        dw, pdw = a.out(dm2, (n,), np.float32)
        self._check(_lib.darbs_cuda_eval(self._h, C.byref(kernel), n, p, pw, pdw, int(exact), a.space))
        return w, dw

    # ---------------------------------------------------------- rasterizer
    def bin(self, mu2, conic, radius, depth, width: int, height: int):
        """bin_splats, src/rasterizer.cpp:25-53."""
        a = _Args()
        n = int(depth.numel() if _is_torch(depth) else np.asarray(depth).size)
        pm, pc = a.ptr(mu2, np.float32, 2 * n), a.ptr(conic, np.float32, 3 * n)
        pr, pd = a.ptr(radius, np.float32, n), a.ptr(depth, np.float32, n)
        tiles = ((width + 15) // 16) * ((height + 15) // 16)
        k = C.c_int64(0)
        space = a.space if a.space is not None else HOST
        # first call: sizes only
        self._check(_lib.darbs_cuda_bin(self._h, n, pm, pc, pr, pd, width, height, C.byref(k), None, None,
                                        None, None, 0, space))
        kk = int(k.value)
        ranges, p_ranges = a.out(depth, (max(tiles, 1), 2), np.int32)
        plist, p_plist = a.out(depth, (max(kk, 1),), np.int32)
        keys, p_keys = a.out(depth, (max(kk, 1),), np.uint64)
        order, p_order = a.out(depth, (max(n, 1),), np.int32)
        self._check(_lib.darbs_cuda_bin(self._h, n, pm, pc, pr, pd, width, height, C.byref(k), p_ranges,
                                        p_plist, p_keys, p_order, kk, space))
        return dict(num_entries=kk, tile_ranges=ranges[:tiles], point_list=plist[:kk], sort_keys=keys[:kk],
                    depth_order=order[:n])

    def forward(self, kernel: KernelSpec, mu2, conic, radius, depth, opacity, rgb, width: int, height: int,
                background, aux: bool = True, image=None):
        """forward, src/rasterizer.cpp:55-112."""
        a = _Args()
        n = int(depth.numel() if _is_torch(depth) else np.asarray(depth).size)
        pm, pc = a.ptr(mu2, np.float32, 2 * n), a.ptr(conic, np.float32, 3 * n)
        pr, pd = a.ptr(radius, np.float32, n), a.ptr(depth, np.float32, n)
        po, pg = a.ptr(opacity, np.float32, n), a.ptr(rgb, np.float32, 3 * n)
        bg = (C.c_float * 3)(*[float(x) for x in background])
        if image is None:
            image, p_img = a.out(depth, (height, width, 3), np.float32)
        else:
            p_img = a.inout(image, np.float32, 3 * width * height)
        out = dict(image=image)
        p_t = p_p = p_c = None
        skipped = C.c_int32(0)
        if aux:
            out["t_final"], p_t = a.out(depth, (height, width), np.float32)
            out["processed"], p_p = a.out(depth, (height, width), np.int32)
            out["contributors"], p_c = a.out(depth, (height, width), np.int32)
        space = a.space if a.space is not None else HOST
        self._check(_lib.darbs_cuda_forward(self._h, C.byref(kernel), n, pm, pc, pr, pd, po, pg, width, height,
                                            bg, p_img, p_t, p_p, p_c, C.byref(skipped) if aux else None, space))
        if aux:
            out["skipped"] = int(skipped.value)
        return out

    def backward(self, kernel: KernelSpec, grad_image, n: int, mu2=None, conic=None, opacity=None, rgb=None,
                 grads=None):
        """backward, src/rasterizer.cpp:147-234; grads[n, 9] in SplatGrads order."""
        a = _Args()
        if _is_torch(grad_image):
            gh, gw = int(grad_image.shape[0]), int(grad_image.shape[1])
        else:
            grad_image = np.ascontiguousarray(grad_image, dtype=np.float32)
            gh, gw = grad_image.shape[0], grad_image.shape[1]
        pgi = a.ptr(grad_image, np.float32)
        pm = a.ptr(mu2, np.float32)
        pc = a.ptr(conic, np.float32)
        po = a.ptr(opacity, np.float32)
        pg = a.ptr(rgb, np.float32)
        if grads is None:
            grads, p_out = a.out(grad_image, (max(n, 1), 9), np.float32)
        else:
            p_out = a.inout(grads, np.float32, 9 * n)
        self._check(_lib.darbs_cuda_backward(self._h, C.byref(kernel), gw, gh, pgi, n, pm, pc, po, pg, p_out,
                                             a.space))
        return grads[:n]

    # ------------------------------------------------------------ geometry
    def realize(self, raw):
        a = _Args()
        n = (raw.numel() if _is_torch(raw) else np.asarray(raw).size) // 14
        p = a.ptr(raw, np.float32, 14 * n)
        prims, pp = a.out(raw, (n, 14), np.float32)
        self._check(_lib.darbs_cuda_realize(self._h, n, p, pp, a.space))
        return prims

    def project(self, kernel: KernelSpec, psi: float, prims, camera, dilation: float = 0.3):
        """project_primitive, src/geometry.cpp:66-87."""
        a = _Args()
        n = (prims.numel() if _is_torch(prims) else np.asarray(prims).size) // 14
        p = a.ptr(prims, np.float32, 14 * n)
        cam, pcam = _cam(camera)
        valid, pv = a.out(prims, (n,), np.int32)
        mu2, pm = a.out(prims, (n, 2), np.float32)
        cov2, pcv = a.out(prims, (n, 3), np.float32)
        conic, pc = a.out(prims, (n, 3), np.float32)
        radius, pr = a.out(prims, (n,), np.float32)
        depth, pd = a.out(prims, (n,), np.float32)
        self._check(_lib.darbs_cuda_project(self._h, C.byref(kernel), psi, dilation, n, p, pcam, pv, pm, pcv, pc,
                                            pr, pd, a.space))
        return dict(valid=valid, mu2=mu2, cov2=cov2, conic=conic, radius=radius, depth=depth)

    def backward_projection(self, psi: float, grad_cov2, grad_mu2, prims, camera):
        """backward_projection, src/geometry.cpp:111-168."""
        a = _Args()
        n = (prims.numel() if _is_torch(prims) else np.asarray(prims).size) // 14
        pgc, pgm = a.ptr(grad_cov2, np.float32, 4 * n), a.ptr(grad_mu2, np.float32, 2 * n)
        p = a.ptr(prims, np.float32, 14 * n)
        cam, pcam = _cam(camera)
        d_mu, p1 = a.out(prims, (n, 3), np.float32)
        d_scale, p2 = a.out(prims, (n, 3), np.float32)
        d_rot, p3 = a.out(prims, (n, 4), np.float32)
        self._check(_lib.darbs_cuda_backward_projection(self._h, psi, n, pgc, pgm, p, pcam, p1, p2, p3, a.space))
        return d_mu, d_scale, d_rot

    # ------------------------------------------------------------ training
    def evaluate_view(self, kernel: KernelSpec, psi: float, raw_params, camera, background=(0.0, 0.0, 0.0),
                      target=None, lam: float = 0.0, grad_image=None, param_grads=None, image_out=None,
                      want_loss: bool = True, accumulate: bool = True):
        """One view of fit_scene's evaluate, src/fit3d.cpp:108-159.  Returns (total, l1, dssim, mse).
        accumulate=False overwrites param_grads instead of adding to it (the first view of an
        iteration: fit3d.cpp:107's fill without the pass that zeroes the array)."""
        if not accumulate:
            self._check(_lib.darbs_cuda_set_accumulate(self._h, 0))
        a, ai = _Args(), _Args()  # parameters and images may live in different spaces
        n = (raw_params.numel() if _is_torch(raw_params) else np.asarray(raw_params).size) // 14
        cam, pcam = _cam(camera)
        w, h = int(cam[4]), int(cam[5])
        p_raw = a.ptr(raw_params, np.float32, 14 * n)
        p_t = ai.ptr(target, np.float32, 3 * w * h)
        p_g = ai.ptr(grad_image, np.float32, 3 * w * h)
        p_pg = a.inout(param_grads, np.float32, 14 * n)
        p_img = ai.inout(image_out, np.float32, 3 * w * h)
        bg = (C.c_float * 3)(*[float(x) for x in background])
        loss = (C.c_double * 4)()
        self._check(_lib.darbs_cuda_evaluate_view(self._h, C.byref(kernel), psi, n, p_raw, pcam, bg, p_t, lam,
                                                  p_g, p_pg, p_img, loss if want_loss else None, a.space,
                                                  ai.space if ai.space is not None else a.space))
        return tuple(float(x) for x in loss)

    def prefetch_target(self, host_image):
        """Start uploading a (pinned) host target image for a later evaluate_view(target=host_image)."""
        if not (isinstance(host_image, np.ndarray) and host_image.dtype == np.float32 and host_image.flags.c_contiguous):
            raise TypeError("prefetch_target needs a contiguous float32 numpy array (same object as the later target)")
        self._check(_lib.darbs_cuda_prefetch_target(self._h, C.c_void_p(host_image.ctypes.data), host_image.size))

    def pop_loss(self):
        """(total, l1, dssim, mse) of the oldest evaluate_view called with want_loss=False."""
        loss = (C.c_double * 4)()
        self._check(_lib.darbs_cuda_pop_loss(self._h, loss))
        return tuple(float(x) for x in loss)

    def loss_total(self, rendered, target, lam: float, want_grad: bool = True):
        """loss_total, src/loss.cpp:173-230.  Images are (h, w, 3).  Returns ((total, l1, dssim, mse), grad)."""
        a = _Args()
        h, w = int(rendered.shape[0]), int(rendered.shape[1])
        pr, pt = a.ptr(rendered, np.float32, 3 * w * h), a.ptr(target, np.float32, 3 * w * h)
        grad, pg = a.out(rendered, (h, w, 3), np.float32) if want_grad else (None, None)
        loss = (C.c_double * 4)()
        self._check(_lib.darbs_cuda_loss_total(self._h, w, h, pr, pt, float(lam), loss, pg, a.space))
        return tuple(float(x) for x in loss), grad

    # ------------------------------------------------------------ multi-GPU (view-parallel)
    def comm_init(self, comm_id: bytes, rank: int, world: int):
        """ncclCommInitRank on this context's GPU (collective over the ranks); comm_id from comm_unique_id()."""
        self._check(_lib.darbs_cuda_comm_init(self._h, comm_id, rank, world))

    def comm_destroy(self):
        self._check(_lib.darbs_cuda_comm_destroy(self._h))

    def allreduce_adam_step(self, params, grads, m, v, lrs, t: int):
        """All-reduce of the gradients over the communicator (if any), then Adam step t; CUDA tensors."""
        ptr = lambda a: C.c_void_p(a.data_ptr())  # noqa: E731
        self._check(_lib.darbs_cuda_allreduce_adam_step(self._h, params.numel(), ptr(params), ptr(grads), ptr(m), ptr(v),
                                                        ptr(lrs), t))

    def train_step(self, kernel: KernelSpec, psi: float, params, grads, m, v, lrs, cameras, targets, lam: float,
                   t: int, n_views_total: int, background=(0.0, 0.0, 0.0), want_loss: bool = True):
        """One fit_scene iteration (src/fit3d.cpp:104-184) over this rank's views: evaluate, all-reduce of the
        gradients over the communicator (if any), Adam.  All arrays are CUDA tensors; cameras: [views][22]."""
        n = params.numel() // 14
        cams = np.ascontiguousarray(np.asarray(cameras, dtype=np.float64).reshape(-1))
        nv = cams.size // 22
        assert nv == len(targets)
        tp = (C.c_void_p * max(nv, 1))(*[C.c_void_p(tt.data_ptr()) for tt in targets])
        bg = (C.c_float * 3)(*[float(x) for x in background])
        loss = (C.c_double * 4)()
        ptr = lambda a: C.c_void_p(a.data_ptr())  # noqa: E731
        self._check(_lib.darbs_cuda_train_step(self._h, C.byref(kernel), psi, n, ptr(params), ptr(grads), ptr(m), ptr(v),
                                               ptr(lrs), nv, cams.ctypes.data_as(C.POINTER(C.c_double)), tp, lam, bg, t,
                                               n_views_total, loss if want_loss else None))
        return tuple(float(x) for x in loss) if want_loss else None

    def adam_step(self, params, grads, m, v, lrs, t: int):
        """adam_step, include/darbs/optim.hpp:24-39 (in place)."""
        a = _Args()
        dim = params.numel() if _is_torch(params) else np.asarray(params).size
        pp, pg = a.inout(params, np.float32, dim), a.ptr(grads, np.float32, dim)
        pm, pv, pl = a.inout(m, np.float32, dim), a.inout(v, np.float32, dim), a.ptr(lrs, np.float32, dim)
        self._check(_lib.darbs_cuda_adam_step(self._h, dim, pp, pg, pm, pv, pl, int(t), a.space))
