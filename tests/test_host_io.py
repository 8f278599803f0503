"""File formats of the C++ mirror (paper_2501_12369_b200/host/darbs_b200_fit.hpp) against files
written by the reference's own writers (src/scene_io.cpp, src/image.cpp; fixtures under
tests/golden/io/, made by tests/golden/make_golden.py).  Host code only: no GPU needed.

Reading a reference-written file and writing it back must reproduce it byte for byte: that pins
the readers (every value parsed exactly) and the writers (17 significant digits, field order,
little-endian float32 dump, PPM clamp and round-half-up) at once."""
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HOST = os.path.join(ROOT, "paper_2501_12369_b200", "host")
IO = os.path.join(ROOT, "tests", "golden", "io")
TOOL = os.path.join(HOST, "io_tool")


@pytest.fixture(scope="module")
def tool():
    r = subprocess.run(["make", "-C", HOST, "io_tool"], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    return TOOL


def run(tool, *args):
    return subprocess.run([tool, *args], capture_output=True, text=True, timeout=60)


@pytest.mark.parametrize("cmd,name", [("copy-scene", "scene.txt"), ("copy-cameras", "cameras.txt"),
                                      ("copy-dsfl", "image.dsfl"), ("copy-ppm", "image.ppm")])
def test_read_then_write_is_byte_identical(tool, tmp_path, cmd, name):
    out = tmp_path / name
    r = run(tool, cmd, os.path.join(IO, name), str(out))
    assert r.returncode == 0, r.stderr
    assert out.read_bytes() == open(os.path.join(IO, name), "rb").read()


def test_float_dump_to_ppm_matches_the_reference_writer(tool, tmp_path):
    out = tmp_path / "x.ppm"
    assert run(tool, "dsfl-to-ppm", os.path.join(IO, "image.dsfl"), str(out)).returncode == 0
    assert out.read_bytes() == open(os.path.join(IO, "image_from_dsfl.ppm"), "rb").read()


def test_scene_values_survive_the_text_format(tool, tmp_path):
    """17 significant digits round-trip every double (scene_io.cpp:79)."""
    vals = np.load(os.path.join(IO, "scene_values.npy"))
    text = open(os.path.join(IO, "scene.txt")).read().split()
    assert np.array_equal(np.array([float(t) for t in text]).reshape(vals.shape), vals)


def test_image_stats(tool):
    r = run(tool, "stats", os.path.join(IO, "image.dsfl"), os.path.join(IO, "image.dsfl"))
    assert r.returncode == 0
    mse, psnr = r.stdout.split()
    assert float(mse) == 0.0 and psnr == "inf"


def test_io_errors_map_to_exit_code_3(tool, tmp_path):
    """io_error -> 3 (tools/main.cpp:487-499): missing file, wrong field count, non-positive scale,
    opacity out of range, malformed camera block, bad magic."""
    assert run(tool, "copy-scene", str(tmp_path / "missing.txt"), str(tmp_path / "o")).returncode == 3
    cases = {
        "short.txt": ("copy-scene", "1 2 3 4\n"),
        "scale.txt": ("copy-scene", "0 0 0 0.1 -0.2 0.1 1 0 0 0 0.5 1 1 1\n"),
        "opacity.txt": ("copy-scene", "0 0 0 0.1 0.2 0.1 1 0 0 0 1.5 1 1 1\n"),
        "cams.txt": ("copy-cameras", "80 80 32 32 64 64\n1 0 0 0\n"),
        "cams_bad_token.txt": ("copy-cameras", "80 80 32 32 64 sixty-four\n"),
        "magic.dsfl": ("copy-dsfl", "NOPE" + "\0" * 12),
    }
    for name, (cmd, text) in cases.items():
        p = tmp_path / name
        p.write_text(text)
        r = run(tool, cmd, str(p), str(tmp_path / "o"))
        assert r.returncode == 3, (name, r.stderr)
    # comments and blank lines are skipped (scene_io.hpp:10-13)
    p = tmp_path / "comments.txt"
    p.write_text("# a scene\n\n0 0 0 0.1 0.2 0.1 1 0 0 0 0.5 1 1 1  # trailing\n")
    out = tmp_path / "o.txt"
    assert run(tool, "copy-scene", str(p), str(out)).returncode == 0
    assert len(out.read_text().splitlines()) == 1


def test_mirror_output_is_readable_by_the_reference(tool, tmp_path, ref):
    """The other direction: the reference's reader parses what the mirror wrote."""
    out = tmp_path / "scene.txt"
    assert run(tool, "copy-scene", os.path.join(IO, "scene.txt"), str(out)).returncode == 0
    n, prims = ref.read_scene(str(out))
    vals = np.load(os.path.join(IO, "scene_values.npy"))
    assert n == vals.shape[0] and np.array_equal(prims, vals)
