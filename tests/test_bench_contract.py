"""The committed bench lines carry the keys the driver and the judge read
(bench contract: metric/value/unit, e2e, roofline, cpu_baseline, clocks,
gpu_launches); checked on the round's recorded output, no GPU needed."""

import json
import os

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def load(name):
    path = os.path.join(ROOT, "profiles", name)
    if not os.path.exists(path):
        pytest.skip(f"{name} not recorded")
    with open(path) as f:
        return json.loads(f.read().strip().splitlines()[-1])


def test_gpu_bench_line_keys():
    b = load("r1_bench_c2.json")
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "e2e", "roofline", "cpu_baseline", "clocks",
              "gpu_launches"):
        assert k in b, k
    assert b["warmup"] >= 3 and b["gpu_launches"] == b["steps"]
    assert b["e2e"]["h2d_bytes_per_step"] > 0 and b["e2e"]["d2h_bytes_per_step"] > 0
    r = b["roofline"]
    assert r["bound"] in ("hbm", "tensor") and 0.0 < r["frac"] < 1.0
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    assert r["traffic"] is None or r["traffic"] > 0
    assert b["cpu_baseline"]["kind"] in ("port", "reference") and b["cpu_baseline"]["cores"] >= 1
    assert not set(b["clocks"]["reasons"]) & {"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"}
    assert "workload" in b["config"] and "model" not in b["config"]


def test_reference_arm_line_keys():
    b = load("r1_bench_reference_c2.json")
    assert b["impl"] == "reference"
    assert b["e2e"]["value"] == b["value"] and b["cpu_baseline"]["value"] == b["value"]
    assert b["metric"] == load("r1_bench_c2.json")["metric"]
