"""bench.py keeps the driver's contract: one JSON line with the required
keys, on short runs of the default mode (config 4 shape, few cameras and
frames), the per-frame mode (config 2) and the reference arm."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REQUIRED = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
            "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "roofline",
            "clocks", "gpu_launches", "e2e"}


def run_bench(*args):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args],
                         capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


def _check_roofline(r):
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and 0 < r["frac"] < 1.2
    assert r["achieved"] > 0 and r["peak"] > 0


def test_bench_default_line_is_config4():
    d = run_bench("--cams", "4", "--frames", "10", "--steps", "4", "--warmup", "3",
                  "--e2e-steps", "1")
    assert REQUIRED <= set(d)
    assert "configs[3]" in d["config"]["workload"]
    assert d["value"] > 0 and d["n_gpus"] == 1 and d["steps"] == 4 and d["warmup"] == 3
    _check_roofline(d["roofline"])
    assert d["e2e"]["value"] > 0 and d["e2e"]["h2d_bytes_per_step"] > 0
    assert d["gpu_launches"] == 4 * 4
    assert "sm_mhz" in d["clocks"] and "reasons" in d["clocks"]
    assert "k1b" in d["mask_path"]
    cb = d["cpu_baseline"]
    assert cb["value"] > 0 and cb["cores"] >= 1 and cb["lscpu_model"]
    sec = d["secondary"]["cfg2"]
    assert sec["value"] > 0 and "configs[1]" in sec["workload"]
    _check_roofline(sec["roofline"])


def test_bench_cfg2_line():
    d = run_bench("--config", "cfg2", "--frames", "10", "--steps", "4", "--warmup", "3", "--no-cpu")
    assert REQUIRED <= set(d)
    _check_roofline(d["roofline"])
    assert d["e2e"]["value"] > 0 and d["gpu_launches"] == 12
    assert d["mask_path"]["mask_fused_launches"] > 0


def test_bench_reference_arm_line():
    d = run_bench("--impl", "reference", "--cams", "2", "--frames", "4", "--steps", "1",
                  "--warmup", "1")
    assert d["impl"] == "reference" and d["value"] > 0
    assert d["config"]["frames_per_step"] == 8
    assert d["cpu_baseline"]["cores"] >= 1 and d["e2e"]["h2d_bytes_per_step"] == 0
