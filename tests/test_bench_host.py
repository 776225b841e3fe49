"""bench.py's host logic, without a GPU: the roofline numerators (algorithmic bytes
and flops per matvec) against the figures SURVEY.md §8 computes independently
from BASELINE.json's configs, and the reference arm's JSON line."""
import json
import os
import subprocess
import sys

import pytest

from gen.hgen import CONFIGS, EXTRA_CONFIGS

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


@pytest.mark.parametrize("name,v_bytes", [("c1", 2.36e6), ("c2", 2.82e9), ("c3", 18.79e9), ("c4", 57.98e9)])
def test_factor_panel_bytes_match_survey(name, v_bytes):
    """V bytes 2.36 MB / 2.82 GB / 18.79 GB / 57.98 GB (C1..C4);
    project streams V once plus x, expand U once plus D plus x and y."""
    cfg = CONFIGS[name]
    ab = bench.alg_bytes(cfg, cfg.N, 1)
    v = ab["project"] - 8 * cfg.N
    assert abs(v - v_bytes) <= 0.005 * v_bytes
    assert ab["expand"] - 16 * cfg.N == v + 8 * cfg.N * cfg.b
    assert ab["factor"] == cfg.factor_bytes        # N (2 (c-1) r L + b) doubles


def test_c4_total_and_dense_bytes():
    """BASELINE configs[3] '~125 GB'; dense D = 8.59 GB (6.9 % of the bytes)."""
    cfg = CONFIGS["c4"]
    ab = bench.alg_bytes(cfg, cfg.N, 1)
    assert abs(ab["factor"] / 1e9 - 124.55) < 0.01
    d = 8 * cfg.N * cfg.b
    assert abs(d / 1e9 - 8.59) < 0.01 and abs(d / ab["factor"] - 0.069) < 0.001


def test_c5_flops_match_survey():
    """618.5 GFLOP per 64-rhs matvec (2 nrhs N (2WL + b))."""
    cfg = CONFIGS["c5"]
    fl = bench.alg_flops(cfg, cfg.N, cfg.nrhs)
    assert abs((fl["project"] + fl["expand"]) / 1e9 - 618.5) < 0.1


def test_standard_levels_counted_from_two():
    """Standard admissibility: level 1 has no admissible pair, so
    the algorithmic bytes count levels 2..L only, with 3^d dense blocks per row."""
    cfg = EXTRA_CONFIGS["s2"]
    ab = bench.alg_bytes(cfg, cfg.N, 1)
    assert ab["factor"] == 8 * cfg.N * (2 * cfg.W * (cfg.L - 1) + 9 * cfg.b)


def test_reference_arm_json_line():
    """`bench.py --impl reference` (the oracle timed on the host) prints one JSON
    line with the contract's keys, on the arm's metric and config."""
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                          "--warmup", "3", "--config", "c1"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["metric"] == bench.METRIC and line["unit"] == "matvec/s"
    assert line["value"] > 0 and line["higher_is_better"] is True and line["n_gpus"] == 1
    assert line["cpu_baseline"]["kind"] == "oracle" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["d2h_bytes_per_step"] == 0
    assert line["config"]["workload"].startswith("c1")


def _clean_env():
    return {k: v for k, v in os.environ.items()
            if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "LOCAL_WORLD_SIZE", "MASTER_ADDR", "MASTER_PORT")}


@pytest.mark.parametrize("n", [2, 4])
def test_gpus_n_starts_n_ranks(n):
    """`python bench.py --gpus N` outside torch.distributed re-executes itself
    under torch.distributed.run with N ranks: every rank sees WORLD_SIZE = N
    and ranks 0..N-1 all report (gloo, host only)."""
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", str(n), "--launcher-check"],
                         capture_output=True, text=True, timeout=300, cwd=ROOT, env=_clean_env())
    assert out.returncode == 0, out.stderr[-3000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["launcher_check"] and line["gpus"] == n and line["world"] == n
    assert line["ranks"] == list(range(n)) and line["worlds"] == [n]


def test_world_size_mismatch_is_an_error():
    """Under a launcher whose world differs from --gpus, bench.py refuses (rc 2)
    instead of silently measuring another GPU count."""
    env = _clean_env()
    env.update(WORLD_SIZE="2", RANK="0", LOCAL_RANK="0")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "4", "--launcher-check"],
                         capture_output=True, text=True, timeout=300, cwd=ROOT, env=env)
    assert out.returncode == 2 and "WORLD_SIZE=2" in out.stderr


def test_reference_arm_same_config_and_sample_as_cpu_baseline():
    """Both CPU-oracle legs use one sample of the workload, and the reference
    arm's `config` is exactly the GPU arm's (same keys and values)."""
    cfg = CONFIGS["c4"]
    q, n, depth, fb = bench.oracle_sample(cfg)
    assert (q, n, depth) == (3, cfg.N // 64, 6) and fb <= bench.SAMPLE_BYTES
    assert bench.workload_config(cfg)["factor_bytes"] == cfg.factor_bytes
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "2",
                          "--warmup", "1", "--config", "c2"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["config"] == json.loads(json.dumps(bench.workload_config(CONFIGS["c2"])))
    assert "leading level-1 diagonal sub-H-matrix of c2" in line["cpu_baseline"]["sample"]


def test_clock_sampler_reports_throttle_reasons_and_power():
    """The clocks object of a bench line from nvidia-smi's CSV samples (the
    ClockSampler query's column order): median SM clock, the throttle reasons
    seen in any sample, median board power, the enforced limit."""
    class _Proc:
        def terminate(self):
            pass

        def wait(self, timeout=None):
            pass

    class _Thread:
        def join(self, timeout=None):
            pass

    cs = bench.ClockSampler(0)
    cs.proc, cs.t = _Proc(), _Thread()
    assert cs.Q.split(",")[3] == "power.draw" and cs.Q.split(",")[9] == "power.limit"
    cs.lines = ["0, 1500, 1965, 998.5, 0x4, Not Active, Not Active, Not Active, Active, 1000.00",
                "0, 1540, 1965, 1001.5, 0x0, Not Active, Not Active, Not Active, Not Active, 1000.00",
                "0, 1520, 1965, 990.0, 0x4, Not Active, Not Active, Not Active, Active, 1000.00",
                "garbage"]
    clk = cs.stop()
    assert clk["sm_mhz"] == 1520.0 and clk["sm_max_mhz"] == 1965.0 and clk["samples"] == 3
    assert clk["reasons"] == ["sw_power_cap"]
    assert clk["power_w"] == 998.5 and clk["power_limit_w"] == 1000.0
