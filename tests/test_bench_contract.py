"""bench.py keeps the driver's JSON-line contract: the reference arm (the oracle on host cores,
CPU) and a short run of our arm (GPU).  Guards against a bench that crashes before printing."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
        "vs_baseline", "dtype", "data", "config", "e2e", "cpu_baseline")


def _line(args, timeout):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                       timeout=timeout, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.strip().splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


def test_reference_arm_line():
    d = _line(["--impl", "reference", "--steps", "2", "--warmup", "1"], 900)
    assert d["impl"] == "reference"
    assert d["steps"] == 2 and d["warmup"] == 1          # K timed steps after W untimed ones
    for k in KEYS:
        assert k in d, k
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["value"] > 0 and d["higher_is_better"] is False


@pytest.mark.gpu
def test_our_arm_line_short():
    d = _line(["--steps", "5", "--warmup", "3", "--n-cand", "16", "--search-cand", "8", "--no-cpu"], 900)
    for k in KEYS + ("roofline", "gpu_launches", "clocks"):
        assert k in d, k
    assert d["value"] > 0 and d["e2e"]["value"] > 0 and d["gpu_launches"] == 5
    assert d["roofline"]["frac"] > 0 and d["roofline"]["peak"] > 0
    assert d["profiling"]["candidates"] == 16
