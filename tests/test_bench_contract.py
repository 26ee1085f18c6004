"""bench.py output contract (the driver parses one JSON line per run).

CPU: the reference arm (`--impl reference`, the oracle on the host cores) on the toy config.
GPU: our arm on the toy config — roofline, cpu_baseline, e2e, gpu_launches and clocks present."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
             "scaling", "vs_baseline", "dtype", "data", "config", "e2e"}


def _run(args, timeout=600):
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, capture_output=True, text=True,
                       timeout=timeout, cwd=ROOT)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [x for x in p.stdout.splitlines() if x.strip().startswith("{")]
    assert len(lines) == 1, p.stdout
    return json.loads(lines[0])


def test_reference_arm_contract():
    d = _run(["--impl", "reference", "--config", "toy", "--steps", "3", "--warmup", "3"])
    assert BASE_KEYS <= set(d), BASE_KEYS - set(d)
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["warmup"] >= 3 and d["steps"] == 3
    assert "workload" in d["config"]
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["value"] == d["value"] and cb["sample"]
    e = d["e2e"]
    assert e["value"] == d["value"] and e["h2d_bytes_per_step"] == 0 and e["d2h_bytes_per_step"] == 0


def test_warmup_floor():
    d = _run(["--impl", "reference", "--config", "toy", "--steps", "2", "--warmup", "1"])
    assert d["warmup"] >= 3


@pytest.mark.gpu
def test_our_arm_contract_toy():
    d = _run(["--config", "toy", "--steps", "4", "--warmup", "3", "--e2e-steps", "2"])
    assert BASE_KEYS <= set(d), BASE_KEYS - set(d)
    assert d["n_gpus"] == 1 and d["value"] > 0 and d["gpu_launches"] > 0
    r = d["roofline"]
    assert r["bound"] in ("hbm", "tensor") and r["peak"] > 0 and r["unit"] in ("GB/s", "TFLOP/s")
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-3
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["value"] > 0
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert "clocks" in d


@pytest.mark.gpu
def test_our_arm_modes_toy():
    """The Q4G64 and attention stand-in modes keep the contract and label themselves."""
    d = _run(["--config", "toy", "--steps", "3", "--warmup", "3", "--e2e-steps", "1", "--weights", "q4",
              "--no-cpu-baseline"])
    assert d["value"] > 0 and d["config"]["weights"] == "q4" and d["dtype"] != "bf16"
    d = _run(["--config", "toy", "--steps", "3", "--warmup", "3", "--e2e-steps", "1", "--attention", "300",
              "--no-cpu-baseline"])
    a = d["config"]["attention"]
    assert d["value"] > 0 and a["kv_positions"] == 300 and a["us_per_layer"] > 0
