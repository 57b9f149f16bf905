"""bench.py keeps the driver contract (one JSON line with the required keys)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, env=None, timeout=900):
    e = dict(os.environ)
    e.update(env or {})
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, capture_output=True, text=True,
                       cwd=ROOT, env=e, timeout=timeout)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
             "vs_baseline", "dtype", "data", "config", "e2e"}


def test_reference_arm_is_the_oracle_on_host_cores():
    d = _run(["--impl", "reference", "--steps", "2", "--warmup", "1"], env={"RK_REF_TOTAL_SECONDS": "2"})
    assert BASE_KEYS <= set(d) and d["impl"] == "reference"
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["value"] == d["value"] > 0
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    assert d["config"]["workload"].startswith("C4")


@pytest.mark.gpu
def test_bench_line_on_gpu():
    d = _run(["--steps", "5", "--warmup", "3", "--no-cpu-baseline", "--no-no-reduce-check", "--e2e-steps", "3"])
    assert BASE_KEYS <= set(d) and d["value"] > 0 and d["n_gpus"] == 1 and d["warmup"] >= 3
    r = d["roofline"]
    assert {"bound", "achieved", "peak", "unit", "frac", "traffic"} <= set(r)
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])
    # per step: candidate key + pass 1 (memo levels + suffix tables + extremes) + pass 2
    assert d["gpu_launches"] % 5 == 0 and d["gpu_launches"] >= 5 * 3
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
