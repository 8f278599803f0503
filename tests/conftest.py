import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run with -m gpu on the GPU box)")


@pytest.fixture(scope="session")
def port():
    """The plain-C restatement oracle (oracle/darbs_oracle.c)."""
    from oracle import cpu

    return cpu.load("port")


@pytest.fixture(scope="session")
def ref():
    """The reference's own sources (oracle/_ref); absent when never built here."""
    from oracle import cpu

    if not cpu.available("reference"):
        pytest.skip("oracle/_ref/libdarbs_ref.so not built (reference sources absent)")
    return cpu.load("reference")


@pytest.fixture(scope="session", params=["port", "reference"])
def any_oracle(request):
    from oracle import cpu

    if not cpu.available(request.param) and request.param == "reference":
        pytest.skip("oracle/_ref/libdarbs_ref.so not built")
    return cpu.load(request.param)


@pytest.fixture(scope="session")
def darbs():
    import paper_2501_12369_b200 as d

    return d


@pytest.fixture(scope="session")
def ctx(darbs):
    c = darbs.Context(0)
    yield c
    c.close()


def f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def scene_f32(s):
    """The float32 arrays the GPU consumes for an oracle Scene (already f32-representable)."""
    return dict(mu2=f32(s.mu2), conic=f32(s.conic), radius=f32(s.radius), depth=f32(s.depth),
                opacity=f32(s.opacity), rgb=f32(s.rgb))


def rel_err(a, b, floor):
    """The reference's own gradient criterion (tests/test_rasterizer.cpp:242-243)."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    den = np.maximum(np.maximum(np.abs(a), np.abs(b)), floor)
    return np.abs(a - b) / den
