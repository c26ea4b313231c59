"""CPU tier: bench.py's reference arm runs here and prints the contract's JSON line."""

import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference",
                          "--steps", "1", "--warmup", "1"], capture_output=True, text=True,
                         timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
                "cpu_baseline", "e2e"):
        assert key in line, key
    assert line["impl"] == "reference"
    assert line["unit"] == "epochs/s" and line["value"] > 0
    assert line["cpu_baseline"]["kind"] == "port" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0
    assert "workload" in line["config"]


KEYS = ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
        "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e",
        "gpu_launches", "clocks")


def _run_bench(*args):
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), *args], capture_output=True,
                         text=True, timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    return json.loads(out.stdout.strip().splitlines()[-1])


import pytest  # noqa: E402


@pytest.mark.gpu
@pytest.mark.parametrize("config", ["c3", "c5"])
def test_our_arm_json_line(config):
    line = _run_bench("--config", config, "--steps", "3", "--warmup", "3", "--no-cpu-baseline")
    for key in KEYS:
        assert key in line, key
    assert line["value"] > 0 and line["unit"] == "epochs/s" and line["n_gpus"] == 1
    r = line["roofline"]
    assert r["bound"] == "l1_data_pipe" and r["achieved"] > 0 and r["peak"] > 0
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    assert 0 < r["frac"] <= 1.1  # a physical fraction of the data-pipe peak
    assert set(r["kernels"]) == {"K2_forward_dual", "K3_adjoint"}
    assert r["hbm"]["peak"] > 0 and r["hbm"]["compulsory_frac"] < 1.0
    e = line["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert line["gpu_launches"] >= 4 * line["steps"]
    assert "sm_mhz" in line["clocks"] and "workload" in line["config"]


def test_gpus_beyond_visible_devices_fails_clearly():
    """--gpus N starts N ranks itself; with fewer visible GPUs it refuses (rc 2) with a
    one-line JSON reason instead of silently timing one rank."""
    import torch

    n = max(2, torch.cuda.device_count() + 1)
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", str(n), "--steps", "1",
                          "--warmup", "3"], capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert out.returncode == 2, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert "error" in line and line["n_gpus"] == n
