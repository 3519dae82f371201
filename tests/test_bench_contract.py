"""bench.py's JSON line carries every key of the driver contract (run on a
small config so the test takes seconds; the C4 numbers live in profiles/)."""

import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _line(args):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args],
                         capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    return json.loads(out.stdout.strip().splitlines()[-1])


_LINES = {}


def test_bench_line_has_the_contract_keys():
    d = _line(["--config", "C1", "--steps", "4", "--warmup", "3"])
    _LINES["b200"] = d
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
              "roofline", "cpu_baseline", "e2e", "gpu_launches", "clocks"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 4 and d["warmup"] == 3 and d["value"] > 0
    assert d["higher_is_better"] is True and d["dtype"] == "f64" and "workload" in d["config"]
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and 0 < r["frac"] == pytest.approx(
        r["achieved"] / r["peak"])
    assert "traffic" in r
    c = d["cpu_baseline"]
    assert c["kind"] == "port" and c["cores"] == 1 and c["value"] > 0 and c["sample"]
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert e["status"] == "optimal-tolerance"
    assert d["gpu_launches"] > 0
    assert d["clocks"]["samples"] > 0 and "reasons" in d["clocks"]
    sc = d["screen"]                  # flow-screen leg
    assert "error" not in sc, sc
    assert sc["product_us"] > 0 and sc["oracle_set_diff"] == 0 and sc["same_as_first"]
    assert sc["roofline"]["bound"] == "fp64" and 0 < sc["roofline"]["frac"] < 1.2
    assert sc["cpu_baseline"]["value"] > 0


def test_reference_arm_line():
    d = _line(["--impl", "reference", "--config", "C1", "--steps", "3", "--warmup", "3"])
    assert d["impl"] == "reference" and d["value"] > 0
    if "b200" in _LINES:               # the driver's same-config check across the two arms
        assert d["config"] == _LINES["b200"]["config"]
        assert (d["metric"], d["unit"]) == (_LINES["b200"]["metric"], _LINES["b200"]["unit"])
    assert d["cpu_baseline"]["kind"] == "port"
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
