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
    d = _line(["--impl", "reference", "--steps", "2", "--warmup", "1", "--config", "c2"], 900)
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
    for k in KEYS + ("roofline", "gpu_launches", "clocks", "batch8", "stage_roofline", "baselines_ms"):
        assert k in d, k
    assert d["value"] > 0 and d["e2e"]["value"] > 0 and d["gpu_launches"] == 5
    assert d["config"]["workload"].startswith("c4 (configs[3] b1)")          # the largest single-GPU config
    assert d["roofline"]["frac"] > 0 and d["roofline"]["peak"] > 0 and d["roofline"]["bound"] == "hbm"
    assert len(d["stage_roofline"]) == d["config"]["stages"] and all(0 < s["frac"] <= 1 for s in d["stage_roofline"])
    b8 = d["batch8"]
    assert b8["workload"].startswith("c4b8") and b8["value"] > d["value"] and b8["roofline"]["bound"] == "tensor"
    # sequential baseline with single-tenant plans is reported next to the mix-plan one
    assert d["baselines_ms"]["seq_graph_single_tenant_plans"] > 0
    assert d["profiling"]["candidates"] == 16 and 0 < d["profiling"]["frac_of_roofline"] < 1
    assert d["profiling"]["search"]["best_P"] >= 0


@pytest.mark.parametrize("config,sched,expect_us,tol", [
    ("c2", "all_concurrent", 3.86, 0.02), ("c2", "uniform", 4.56, 0.02), ("c3", "all_concurrent", 41.9, 0.05),
    ("c4", "all_concurrent", 48.3, 0.15), ("c4b8", "all_concurrent", 167.3, 0.1)])
def test_stage_roofline_matches_survey_d4(config, sched, expect_us, tol):
    """bench.py's per-stage roofline (max(F_s/TC, B_s/HBM), B_s = stage B_min) at the spec peaks
    reproduces SURVEY §8(d) d.4's derived mix / per-schedule bounds"""
    import numpy as np

    import bench
    from paper_2111_14255_b200 import mt
    from workloads import configs, zoo
    gs = configs.tenants(config)
    L = [g.n_ops for g in gs]
    c = mt.Context(-1)
    c.load_graphs(gs, [[(0x1000, 0x2000, 0x3000) if g.params[j] else None for j in range(g.n_ops)] for g in gs])
    c.set_schedule_pointers({"all_concurrent": configs.all_concurrent_pointers,
                             "uniform": configs.uniform_pointers}[sched](L))
    F, Wb = bench.op_tables(c, gs)
    r = bench.stage_rooflines(np.asarray(c.get_schedule()).tolist(), gs, F, Wb, 2.25e15, 8e12,
                              zoo.make_input(gs[0]).nbytes)
    assert abs(sum(v[0] for v in r) * 1e6 - expect_us) <= tol
