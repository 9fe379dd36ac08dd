"""bench.py keeps its JSON contract (a short run on the GPU): the keys the
driver reads, their units and consistency -- value vs ms_per_step, the
roofline object of the dominant kernel, the e2e object with non-zero copy
bytes, the CPU oracle baseline, clocks, gpu_launches and host_enqueue."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_json_contract():
    cmd = [sys.executable, "bench.py", "--steps", "3", "--warmup", "3", "--frames-per-step", "20",
           "--cpu-seconds", "2"]
    res = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert res.returncode == 0, res.stderr[-3000:]
    line = [x for x in res.stdout.splitlines() if x.startswith("{")][-1]
    d = json.loads(line)
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e", "clocks", "gpu_launches"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3 and d["higher_is_better"] is True
    assert d["unit"] == "frames/s" and d["value"] > 0
    assert abs(d["value"] - 20 / (d["ms_per_step"] / 1e3)) <= 0.01 * d["value"]
    assert "workload" in d["config"] and "l2" in d["config"]
    rl = d["roofline"]
    assert rl["kernel"] == "k_blend_wi" and rl["bound"] == "alu" and rl["unit"] == "T lane-ops/s"
    assert 0 < rl["flop_model"]["frac"] < 1
    assert 0 < rl["frac"] < 1 and abs(rl["frac"] - rl["achieved"] / rl["peak"]) < 1e-3
    assert rl["traffic"] is None or rl["traffic"] > 0
    e2e = d["e2e"]
    assert e2e["unit"] == "frames/s" and 0 < e2e["value"] <= d["value"] * 1.05
    assert e2e["h2d_bytes_per_step"] > 0 and e2e["d2h_bytes_per_step"] >= 20 * 3 * 1352 * 1014 * 4
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["value"] > 0 and cb["cores"] >= 1 and cb["sample"]
    assert d["gpu_launches"] >= 20 * 3 * 18
    assert d["clocks"]["sm_mhz"] is None or d["clocks"]["sm_mhz"] > 0
    assert 0 < d["host_enqueue"]["vs_device"] < 5
