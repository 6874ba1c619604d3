"""bench.py's output contract (the driver parses these lines): the reference
arm on CPU (tiny config, one update) and, on a GPU, the B200 arm's JSON keys
-- value / e2e / roofline / cpu_baseline / clocks / gpu_launches."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _last_json(args, timeout):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT,
                       capture_output=True, text=True, timeout=timeout)
    assert r.returncode == 0, r.stderr[-2000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


def test_reference_arm_contract():
    d = _last_json(["--impl", "reference", "--config", "tiny", "--steps", "1", "--warmup", "0"],
                   300)
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    for k in ("metric", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "scaling", "dtype",
              "data", "config"):
        assert k in d, k
    assert d["cpu_baseline"]["kind"] in ("reference", "port") and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}
    assert d["workers_1"]["value"] > 0 and d["workers_1"]["cores"] == 1
    # the reference arm runs the reference alone: no product library mapped
    assert d["native_so_mapped"] == ["oracle/_ref/libmtkref.so"], d["native_so_mapped"]


@pytest.mark.gpu
def test_b200_arm_contract(cuda):
    d = _last_json(["--config", "tiny", "--steps", "3", "--warmup", "3", "--no-cpu-baseline"], 600)
    assert d["value"] > 0 and d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3
    assert d["higher_is_better"] is True and d["scaling"] == "weak"
    assert "workload" in d["config"]
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    r = d["roofline"]
    assert r["bound"] in ("hbm", "tensor") and r["unit"] in ("GB/s", "TFLOP/s")
    assert 0 < r["frac"] <= 1.0 and abs(r["achieved"] / r["peak"] - r["frac"]) < 1e-3
    assert "traffic" in r
    assert "sm_mhz" in d["clocks"] and "reasons" in d["clocks"]
    assert d["gpu_launches"] > 0
