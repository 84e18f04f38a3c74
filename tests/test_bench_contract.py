"""bench.py's reference arm honours the driver's JSON contract on the CPU
(the GPU arm is exercised by the round-end bench run)."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                          "--warmup", "0", "--n", "64", "--ref-rows", "2"],
                         capture_output=True, text=True, timeout=600, check=True)
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert key in d, key
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    # "reference" when the unmodified reference is installed in baseline/_ref, else the oracle port
    assert d["cpu_baseline"]["kind"] in ("reference", "port") and d["cpu_baseline"]["cores"] >= 1
    assert d["cpu_baseline"]["single_core"]["value"] > 0
    # the line describes what ran, and ms_per_step is one full half step of the configured grid
    assert d["steps"] == 1 and d["warmup"] == 1
    assert abs(d["ms_per_step"] - 1e3 * 64 * 64 * 41 / (d["value"] * 1e9)) <= 1e-9 * d["ms_per_step"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert "workload" in d["config"]
