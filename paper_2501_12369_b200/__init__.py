"""B200-native differentiable DARBF splatting rasterizer.

The product is the CUDA library ``libdarbs_cuda.so`` (sources in ``csrc/``, C ABI in
``include/darbs_cuda.h``) and its C++ mirror of the reference's entry points
(``host/darbs_b200.hpp``).  This Python package is only the ctypes binding the
tests and ``bench.py`` drive that ABI through; PyTorch is used for device
memory, streams and ``torch.distributed`` — plumbing, not the product.

There is NO CPU fallback: importing :mod:`paper_2501_12369_b200.api` raises if the
CUDA library has not been built, and creating a context raises if no B200 is
visible.
"""
from .api import (  # noqa: F401
    DEVICE,
    HOST,
    Context,
    DarbsError,
    KernelSpec,
    default_psi,
    kernel_preset,
    lib_path,
    make_kernel,
    version,
)

__all__ = [
    "Context",
    "DarbsError",
    "KernelSpec",
    "HOST",
    "DEVICE",
    "kernel_preset",
    "make_kernel",
    "default_psi",
    "lib_path",
    "version",
]
