"""The C++ mirror of the reference's entry points (paper_2501_12369_b200/host/darbs_b200.hpp):
its test driver re-runs the closed-form cases of the reference's tests/test_rasterizer.cpp through
darbs::forward / darbs::backward / darbs::bin_splats with the reference's own signatures."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HOST = os.path.join(ROOT, "paper_2501_12369_b200", "host")


def test_host_mirror_builds_against_the_abi():
    """CPU: the header compiles and links against libdarbs_cuda.so with the host compiler alone."""
    r = subprocess.run(["make", "-C", HOST], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    assert os.path.exists(os.path.join(HOST, "test_host"))
    assert os.path.exists(os.path.join(HOST, "test_fit"))


@pytest.mark.gpu
def test_host_mirror_driver():
    if not os.path.exists(os.path.join(HOST, "test_host")):
        subprocess.run(["make", "-C", HOST], check=True, capture_output=True)
    r = subprocess.run([os.path.join(HOST, "test_host")], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "host mirror ok" in r.stdout


@pytest.mark.gpu
def test_host_fit_driver():
    """darbs_b200_fit.hpp: project_primitive / backward_projection / loss_total / adam_step /
    render_scene / fit_scene / fit_image with the reference's signatures, on the cases of its
    tests/test_geometry.cpp, test_loss.cpp and test_fit.cpp."""
    if not os.path.exists(os.path.join(HOST, "test_fit")):
        subprocess.run(["make", "-C", HOST], check=True, capture_output=True)
    r = subprocess.run([os.path.join(HOST, "test_fit")], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "host fit ok" in r.stdout
