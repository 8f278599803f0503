"""B200-native differentiable DARBF splatting rasterizer.

The product is the CUDA library ``libdarbs_cuda.so`` (sources in ``csrc/``, C ABI in
``include/darbs_cuda.h``) and its C++ mirror of the reference's entry points
(``host/darbs_b200.hpp``).  This Python package is only the ctypes binding the
tests and ``bench.py`` drive that ABI through; PyTorch is used for device
memory, streams and ``torch.distributed`` — plumbing, not the product.

There is NO CPU fallback: :mod:`paper_2501_12369_b200.api` (loaded on first use of any name
below) raises if the CUDA library has not been built, and creating a context raises if no B200 is
visible.
"""
_API = ("DEVICE", "HOST", "Context", "DarbsError", "KernelSpec", "comm_unique_id", "default_psi", "kernel_preset",
        "lib_path", "make_kernel", "version")

__all__ = list(_API)


def __getattr__(name):
    """The binding (and with it libdarbs_cuda.so) is loaded on first use of any of its names, so
    that :mod:`paper_2501_12369_b200.synthetic` — pure numpy, the workload generator shared with
    ``bench.py --impl reference`` — can be imported in a process that must not load the product
    library.  Using the product without the built library still raises here."""
    if name in _API or name == "api":
        import importlib

        api = importlib.import_module(".api", __name__)
        return api if name == "api" else getattr(api, name)
    raise AttributeError(f"module {__name__!r} has no attribute {name!r}")
