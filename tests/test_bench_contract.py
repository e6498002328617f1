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
    # every step covers ALL points of the workload (streamed in slabs), so
    # the reference arm's config is our arm's config
    d = _run(["--impl", "reference", "--steps", "2", "--warmup", "1", "--cpu-sample", "4096",
              "--points", str(3 * 4096 + 1000)])
    assert REQUIRED <= set(d)
    assert d["impl"] == "reference" and d["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert d["cpu_baseline"]["kind"] in ("reference", "port")
    sys.path.insert(0, str(ROOT))
    import bench

    assert d["config"] == bench.workload_config(3 * 4096 + 1000, 1)
    assert "3 slabs of 4096 points (+1000)" in d["cpu_baseline"]["sample"]


def test_config_table_is_compact_and_last():
    sys.path.insert(0, str(ROOT))
    import bench

    gpu = {"rows": {"C1_dtg_64^3": {"N": 64**3, "us": 8.1, "frac": 0.87, "pts": 3.2e10,
                                    "us_b2b": 6.4}},
           "floor_us": 2.0, "method": "m"}
    cpu = {"C1_dtg_64^3": {"c": 2.7e8, "c_n": 64**3, "np1": 2.2e7, "np_n": 64**3, "npT": 1e7},
           "host": "16x cpu"}
    line = {"roofline": {"frac": 1.0}, "ms_per_step": 20.5, "value": 1.3e10,
            "cpu_baseline": {"value": 8.5e7}}

    class A:
        points = 1 << 28

    t = bench.config_table(gpu, cpu, line, A)
    assert t["C1_dtg_64^3"] == [262144, 8.1, 0.87, 32000.0, 270.0, 22.0, 10.0, 6.4]
    assert t["cols"][-1] == "gpu_us_b2b"
    assert t["C5_p2_2^28"][:2] == [1 << 28, 20500.0] and t["cpu_host"] == "16x cpu"
    assert t["C5_p2_2^28"][-1] == 20500.0
    assert len(json.dumps(t)) < 2500


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
    link = d["e2e"]["link"]  # the e2e leg's roofline: this box's copy rates
    assert link["h2d_gbs"] > 1 and link["d2h_gbs"] > 1
    assert 0 < link["frac"] <= 1.05 and link["floor_s"] > 0
    assert d["dtype"] == "f64" and d["higher_is_better"] is True
