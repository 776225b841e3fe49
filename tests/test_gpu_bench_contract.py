"""bench.py's JSON line on the GPU (c1, a few steps): every key the driver's
contract names, with consistent values (value = 1000 / ms_per_step, the
roofline fraction = achieved / peak, gpu_launches = the library's count)."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_json_line_contract():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--config", "c1", "--steps", "5",
                          "--warmup", "3"], capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e", "gpu_launches", "clocks"):
        assert k in line, k
    assert line["n_gpus"] == 1 and line["steps"] == 5 and line["warmup"] == 3 and line["dtype"] == "f64"
    assert abs(line["value"] - 1e3 / line["ms_per_step"]) <= 1e-6 * line["value"]
    r = line["roofline"]
    assert r["bound"] in ("hbm", "tensor") and abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    assert line["config"]["workload"].startswith("c1")
    assert line["gpu_launches"] == 2 * line["steps"]                 # project + expand per step
    c = line["cpu_baseline"]
    assert c["kind"] == "oracle" and c["cores"] >= 1 and c["value"] > 0 and c["sample"]
    e = line["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] == 8 * 4096 and e["d2h_bytes_per_step"] == 8 * 4096
    assert "sm_mhz" in line["clocks"] and "reasons" in line["clocks"]
