"""bench.py itself on tiny workloads (one GPU): both configurations run end to end and print one JSON
line with the keys the driver reads.  Guards the driver's round-end bench against a crash in a leg
that the parity tests do not touch (the end-to-end loops, the drop-in timing, configs[3])."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REQUIRED = ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
            "vs_baseline", "dtype", "data", "config", "clocks", "e2e", "gpu_launches", "roofline")


def run_bench(*args):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                       timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


def test_config2_line_on_a_small_scene():
    d = run_bench("--steps", "2", "--splats", "30000", "--width", "480", "--height", "272", "--focal", "400",
                  "--no-cpu-baseline")
    for key in REQUIRED:
        assert key in d, key
    assert d["value"] > 0 and d["e2e"]["value"] > 0 and d["gpu_launches"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 4 * 12 * 480 * 272
    r = d["roofline"]
    for key in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert key in r, key
    assert 1000.0 < r["peak_sm_mhz"] < 2500.0
    assert d["e2e_dropin"]["value"] > 0 and len(d["e2e_dropin"]["small_scene_latency"]) == 2


def test_config3_line_on_a_small_scene():
    d = run_bench("--config", "3", "--views", "3", "--steps", "1", "--splats", "30000", "--width", "480", "--height",
                  "272", "--focal", "400")
    for key in REQUIRED:
        assert key in d, key
    assert d["scaling"] == "strong" and d["config"]["views"] == 3
    assert d["value"] > 0 and d["e2e"]["value"] > 0 and d["e2e"]["losses_read"] == 3 * 4 * 1
