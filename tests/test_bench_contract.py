"""bench.py keeps the driver's JSON-line contract: the reference arm (the reference's own C++
path from oracle/_ref on the host cores, no GPU) and, on a B200, our arm with the roofline,
cpu_baseline, e2e, clocks and gpu_launches objects."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
             "vs_baseline", "dtype", "data", "config", "e2e"}


def run_bench(*args, timeout=600):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT, capture_output=True,
                       text=True, timeout=timeout)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


def test_reference_arm_line():
    line = run_bench("--impl", "reference", "--steps", "3", "--warmup", "3", "--cpu-pairs", "4")
    assert BASE_KEYS <= set(line)
    assert line["impl"] == "reference"
    assert line["metric"] == "scrambled-attn decode tokens/s" and line["unit"] == "tokens/s"
    assert line["value"] > 0 and line["steps"] == 3 and line["warmup"] == 3
    cb = line["cpu_baseline"]
    assert cb["kind"] == "reference" and cb["cores"] >= 1 and cb["value"] == line["value"]
    assert line["e2e"] == {"value": line["value"], "unit": "tokens/s", "h2d_bytes_per_step": 0,
                           "d2h_bytes_per_step": 0}


@pytest.mark.gpu
def test_our_arm_line():
    line = run_bench("--steps", "5", "--warmup", "3", "--no-prefill", "--no-gqa", "--cpu-pairs", "4")
    assert BASE_KEYS <= set(line)
    assert line["n_gpus"] == 1 and line["steps"] == 5 and line["value"] > 0
    assert line["config"]["workload"].startswith("BASELINE cfg2")
    assert line["gpu_launches"] > 0
    e2e = line["e2e"]
    assert 0 < e2e["value"] <= line["value"] * 1.05 and e2e["h2d_bytes_per_step"] > 0 and e2e["d2h_bytes_per_step"] > 0
    rf = line["roofline"]
    assert rf["bound"] == "hbm" and rf["unit"] == "GB/s" and rf["achieved"] > 0 and rf["peak"] > 0
    assert abs(rf["frac"] - rf["achieved"] / rf["peak"]) < 1e-6
    assert line["cpu_baseline"]["kind"] == "reference" and line["cpu_baseline"]["value"] > 0
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(line["clocks"])


@pytest.mark.gpu
def test_prefill_config_line():
    line = run_bench("--config", "3", "--steps", "5", "--warmup", "3")
    assert line["metric"] == "scrambled-attn prefill TFLOP/s" and line["value"] > 0
    assert line["roofline"]["bound"] == "tensor"
    assert 0 < line["e2e"]["value"] <= line["value"] * 1.05
