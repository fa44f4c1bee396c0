"""bench.py's nf arm end to end on the GPU (the driver contract): one JSON line with the
base keys, the device-timed value, the roofline object of the dominant kernel, clocks
sampled during the timed region, an e2e object whose copies are counted, the launch
count and the in-run oracle parity of layer 0.  Run on a
2-layer cut of configs[1] so that it takes seconds (the driver runs the full step)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.gpu
def test_bench_nf_arm_json_contract():
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--layers", "2", "--steps", "3", "--warmup",
                        "3", "--no-cpu-baseline", "--no-ablation"], cwd=ROOT, capture_output=True, text=True,
                       timeout=900)
    assert p.returncode == 0, p.stderr[-3000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, p.stdout[-3000:]
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "clocks", "e2e", "gpu_launches", "parity"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3 and d["dtype"] == "bf16"
    assert d["value"] > 0 and d["ms_per_step"] > 0 and d["higher_is_better"] is True
    rf = d["roofline"]
    assert rf["bound"] in ("hbm", "tensor") and rf["unit"] in ("GB/s", "TFLOP/s")
    assert rf["achieved"] > 0 and rf["peak"] > 0 and abs(rf["frac"] - rf["achieved"] / rf["peak"]) < 1e-6
    assert d["clocks"]["sm_mhz"] > 0 and d["clocks"]["samples"] >= 1
    e2e = d["e2e"]
    assert e2e["value"] > 0 and e2e["h2d_bytes_per_step"] > 0 and e2e["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] > 0
    assert d["parity"]["ok"] is True and d["parity"]["rel_l2"] <= d["parity"]["tolerance"]["rel_l2"]
