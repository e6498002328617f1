"""bench.py keeps the driver contract: one JSON line with the required keys
(reference arm on CPU here; our arm on the GPU)."""

import json
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
REQUIRED = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
            "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "e2e"}


def _run(args, timeout=600):
    res = subprocess.run([sys.executable, str(ROOT / "bench.py"), *args], capture_output=True,
                         text=True, timeout=timeout, cwd=ROOT)
    assert res.returncode == 0, res.stderr[-2000:]
    lines = [ln for ln in res.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1, res.stdout
    return json.loads(lines[0])


def test_reference_arm_line():
    d = _run(["--impl", "reference", "--steps", "2", "--warmup", "1", "--cpu-sample", "4096"])
    assert REQUIRED <= set(d)
    assert d["impl"] == "reference" and d["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert d["cpu_baseline"]["kind"] in ("reference", "port")
    assert isinstance(d["config"], dict) and "workload" in d["config"]


@pytest.mark.gpu
def test_our_arm_line():
    d = _run(["--points", str(1 << 22), "--steps", "3", "--warmup", "3", "--e2e-steps", "1",
              "--cpu-sample", "65536", "--cpu-seconds", "0.5", "--no-configs"])
    assert REQUIRED <= set(d) | {"e2e"}
    assert {"roofline", "cpu_baseline", "clocks", "gpu_launches"} <= set(d)
    r = d["roofline"]
    assert r["bound"] == "hbm" and 0 < r["frac"] < 1.5 and r["unit"] == "GB/s"
    assert d["gpu_launches"] == 3
    assert d["e2e"]["h2d_bytes_per_step"] == 320 * (1 << 22)
    assert d["e2e"]["d2h_bytes_per_step"] == 192 * (1 << 22)
    assert d["dtype"] == "f64" and d["higher_is_better"] is True
