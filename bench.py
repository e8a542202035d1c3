"""Benchmark of the multi-tenant stage executor (BASELINE.json metric: multi-tenant latency ms vs
sequential / multi-stream; schedules profiled / sec).

One step = one mt_run of the whole hot path (input pack + every tenant op of every stage, one
cooperative launch) over one batch of the synthetic workload, inputs resident in HBM.
Default workload = BASELINE.json configs[1]: ResNet-18 + MobileNet-V2, 224x224, batch 1, bf16.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c2]

Multi-GPU (torchrun, one process per GPU): the executor runs as independent replicas (a
schedule's latency is a single-GPU property: DESIGN.md "replicas only"), and the schedule-
profiling leg shards candidates c -> rank c mod N with one NCCL all_gather of the latencies.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from workloads import configs, zoo  # noqa: E402

METRIC = "multi-tenant latency ms vs sequential/multi-stream; schedules profiled/sec"
CONFIG_NAMES = {"c1": "configs[0]", "c2": "configs[1]", "c3": "configs[2]", "c4": "configs[3] b1",
                "c4b8": "configs[3] b8"}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2")
    ap.add_argument("--profile-config", default="c3")
    ap.add_argument("--n-cand", type=int, default=1024)
    ap.add_argument("--search-cand", type=int, default=64)
    ap.add_argument("--no-profile", action="store_true")
    ap.add_argument("--no-baselines", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--warm-l2", action="store_true", help="do not flush L2 between timed steps")
    return ap.parse_args()


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region (B200_PROFILING.md)"""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.p = None

    def __enter__(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "50"],
                                      stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.p = None
        return self

    def _read(self):
        for line in self.p.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.p:
            self.p.terminate()
            try:
                self.p.wait(timeout=2)
            except Exception:
                self.p.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 2 + i and r[2 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# ------------------------------------------------------------------------------------------
# reference arm: the CPU oracle as it stands (the only other place bench.py executes oracle/)
# ------------------------------------------------------------------------------------------
def oracle_sample(config, budget_s=10.0, max_reps=5):
    from oracle import forward as fw
    graphs = configs.tenants(config)
    x = zoo.make_input(graphs[0])
    t0 = time.perf_counter()
    times = []
    while len(times) < max_reps and (time.perf_counter() - t0) < budget_s:
        t1 = time.perf_counter()
        for g in graphs:
            fw.forward(g, x, "bf16")
        times.append(time.perf_counter() - t1)
    try:
        from threadpoolctl import threadpool_info
        cores = max((i.get("num_threads", 1) for i in threadpool_info()), default=1)
    except Exception:
        cores = os.cpu_count()
    return float(np.mean(times)) * 1e3, len(times), cores


def run_reference(args, ws, rank, budget_s=240.0):
    """The tier's reference arm: the CPU oracle as it stands, on the host cores.  W untimed steps,
    then K timed steps; a step = one full multi-tenant forward pass of the workload (all tenants,
    one batch).  If K steps would exceed budget_s the run stops early and says so (steps = done)."""
    if rank != 0:
        return
    from oracle import forward as fw
    cfg = args.config
    graphs = configs.tenants(cfg)
    x = zoo.make_input(graphs[0])

    def step():
        for g in graphs:
            fw.forward(g, x, "bf16")

    for _ in range(args.warmup):
        step()
    times = []
    t0 = time.perf_counter()
    while len(times) < args.steps:
        t1 = time.perf_counter()
        step()
        times.append(time.perf_counter() - t1)
        if time.perf_counter() - t0 + times[-1] > budget_s:
            break
    ms, reps = float(np.mean(times)) * 1e3, len(times)
    try:
        from threadpoolctl import threadpool_info
        cores = max((i.get("num_threads", 1) for i in threadpool_info()), default=1)
    except Exception:
        cores = os.cpu_count()
    line = {"impl": "reference", "metric": METRIC, "value": ms, "unit": "ms", "n_gpus": args.gpus,
            "steps": reps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": False,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{cfg} ({CONFIG_NAMES.get(cfg, cfg)}): " + configs.CONFIGS[cfg][3],
                       "parallelism": "cpu"},
            "cpu_baseline": {"value": ms, "unit": "ms", "cores": cores, "kind": "oracle",
                             "sample": f"{reps} full multi-tenant forward passes (all tenants, batch "
                                       f"{configs.CONFIGS[cfg][1]}), numpy fp64 with bf16 storage emulation"},
            "e2e": {"value": ms, "unit": "ms", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------------------
# our arm
# ------------------------------------------------------------------------------------------
def main():
    args = parse()
    ws, rank, local = dist_env()
    if args.impl == "reference":
        run_reference(args, ws, rank)
        return
    import torch
    import torch.distributed as dist

    from paper_2111_14255_b200.session import TenantMix

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if ws > 1:
        dist.init_process_group("nccl", device_id=dev)
    stream = torch.cuda.current_stream(dev)
    sp = stream.cuda_stream
    K, W = args.steps, max(args.warmup, 3)
    flush = None if args.warm_l2 else torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    def barrier():
        if ws > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    def maxall(v):
        if ws == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def same_knobs(m):
        """measured executor knobs (partition rule, claim depth); every rank uses rank 0's choice
        so latencies stay comparable across ranks"""
        kn, med = m.calibrate()
        if ws > 1:
            t = torch.tensor(list(kn), dtype=torch.int64, device=dev)
            dist.broadcast(t, 0)
            kn = tuple(int(v) for v in t.tolist())
            m.set_knobs(kn)
        return kn, med

    graphs = configs.tenants(args.config)
    L = [g.n_ops for g in graphs]
    mix = TenantMix(graphs, device=local)
    x = zoo.make_input(graphs[0])
    mix.set_input(x)
    ctx = mix.ctx

    def time_steps(fn, steps, warm):
        for _ in range(warm):
            fn()
        barrier()
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
        for a, b in evs:
            if flush is not None:
                flush.fill_(1)
            a.record(stream)
            fn()
            b.record(stream)
        barrier()
        return [a.elapsed_time(b) for a, b in evs]

    # ---- SM-partition rule chosen by measurement (outside the timed region) ----
    knobs, knob_med = same_knobs(mix)
    # ---- schedule search (outside the timed region): profile candidates, keep the best ----
    cands = configs.sample_candidates(L, args.search_cand, seed=14255)
    named = {"all_concurrent": configs.all_concurrent_pointers(L),
             "sequential": configs.sequential_pointers(L),
             "uniform4": configs.uniform_pointers(L)}
    lat, st = ctx.profile_batch_pointers(cands, mix.in_ptrs, mix.out_ptrs, warmup=2, iters=5, stream=sp)
    best = int(np.nanargmin(np.where(st == 0, lat, np.nan)))
    named["best_of_%d" % len(cands)] = cands[best]

    results = {}
    for name, rho in named.items():
        ctx.set_schedule_pointers(rho)
        t = time_steps(lambda: ctx.run_async(mix.in_ptrs, mix.out_ptrs, sp), max(K // 4, 20), W)
        results[name] = float(np.mean(t))
    head_name = min(results, key=results.get)
    ctx.set_schedule_pointers(named[head_name])
    n_stages = ctx.num_stages()

    # ---- headline timed region (clocks sampled throughout) ----
    with ClockSampler(local) as clk:
        t_end = time.time() + 0.4
        while time.time() < t_end:           # bring clocks under load before timing
            ctx.run_async(mix.in_ptrs, mix.out_ptrs, sp)
        step_ms = time_steps(lambda: ctx.run_async(mix.in_ptrs, mix.out_ptrs, sp), K, W)
    ms = maxall(float(np.mean(step_ms)))
    _, stage_us = ctx.run(mix.in_ptrs, mix.out_ptrs, sp)

    # ---- baselines: the same kernels, one launch per op ----
    base = {}
    if not args.no_baselines:
        for mode in ("seq", "seq_graph", "ms_dfs", "ms_bfs", "ms_graph", "stage_events"):
            t = time_steps(lambda: ctx.run_baseline(mode, mix.in_ptrs, mix.out_ptrs, sp), max(K // 4, 20), W)
            base[mode] = maxall(float(np.mean(t)))

    # ---- end-to-end through the C ABI with HOST buffers (pinned), H2D + D2H in the timed region
    xh = torch.from_numpy(x).pin_memory()
    outs_h = [torch.empty(o.shape, dtype=torch.float32).pin_memory() for o in mix.outputs]
    e2e = [ctx.run_host([xh.data_ptr()] * len(L), [o.data_ptr() for o in outs_h], sp) for _ in range(W + K)][W:]
    e2e_ms = maxall(float(np.mean(e2e)) / 1e3)
    h2d = int(x.nbytes)
    d2h = int(sum(o.numel() * 4 for o in outs_h))

    # ---- roofline of the dominant (only) kernel: the executor launch ----
    F = sum(ctx.op_cost(t, j)[0] for t in range(len(L)) for j in range(L[t]))
    B_op = sum(ctx.op_cost(t, j)[1] for t in range(len(L)) for j in range(L[t]))
    wbytes = sum(2 * int(np.prod(p["weight"].shape)) for g in graphs for p in g.params if p and "weight" in p)
    B_min = wbytes + x.nbytes + sum(g.batch * g.out_classes * 4 for g in graphs)
    pk = peaks()
    hbm = pk.get("hbm_gbs", 6650.0)
    tc = pk.get("bf16_tflops", 1590.0)
    t_s = ms * 1e-3
    hbm_bound = B_min / (hbm * 1e9) >= F / (tc * 1e12)
    traffic = None
    try:
        prof = json.load(open(os.path.join(ROOT, "profiles", "r01_executor_ncu.json")))
        traffic = prof.get(args.config, {}).get("dram_bytes_per_launch")
    except Exception:
        pass
    roof = ({"bound": "hbm", "achieved": B_min / t_s / 1e9, "peak": hbm, "unit": "GB/s",
             "frac": B_min / t_s / 1e9 / hbm, "traffic": traffic,
             "algorithmic_bytes": int(B_min), "bytes_op_materialized": int(B_op)}
            if hbm_bound else
            {"bound": "tensor", "achieved": F / t_s / 1e12, "peak": tc, "unit": "TFLOP/s",
             "frac": F / t_s / 1e12 / tc, "traffic": traffic, "algorithmic_flops": int(F)})
    roof["kernel"] = "mtk::executor_kernel (whole step = 1 launch)"
    roof["peak_source"] = "MEASURED_PEAKS.json (burst)" if pk else "B200_PROFILING.md fallback"

    # ---- schedules profiled per second (config 5: candidates of the 3-tenant mix) ----
    prof_line = None
    if not args.no_profile:
        del mix
        torch.cuda.empty_cache()
        pg = configs.tenants(args.profile_config)
        pmix = TenantMix(pg, device=local)
        pmix.set_input(zoo.make_input(pg[0]))
        PL = [g.n_ops for g in pg]
        allc = configs.sample_candidates(PL, args.n_cand, seed=14255)
        from paper_2111_14255_b200 import distributed as D
        pknobs, _ = same_knobs(pmix)
        pfn = lambda cs: pmix.ctx.profile_batch_pointers(cs, pmix.in_ptrs, pmix.out_ptrs, 2, 10, sp)
        pmix.ctx.profile_batch_pointers(allc[:8], pmix.in_ptrs, pmix.out_ptrs, 1, 1, sp)  # warm
        barrier()
        t0 = time.perf_counter()
        pinfo = {}   # N > 1: every rank also times the two extremes (candidates 0, 1) for per-GPU scaling
        lat_all, st_all = D.profile_distributed(pfn, allc, rank, ws, device=dev,
                                                ref=(0, 1) if ws > 1 else None, info=pinfo)
        torch.cuda.synchronize(dev)
        dt = maxall(time.perf_counter() - t0)
        lat_p = lat_all[st_all == 0]
        st_p = st_all
        # Alg.1 coordinate descent on the same mix (P=3, R=1, M=8), rank 0's GPU
        search_line = None
        if rank == 0:
            from paper_2111_14255_b200 import search as search_mod
            t1 = time.perf_counter()
            cdr = search_mod.coordinate_descent(pfn, PL, P=3, rounds=1, m=8, seed=14255)
            search_line = {"algorithm": "coordinate descent (Alg.1), P=3 R=1 M=8", "evaluations": cdr.evaluations,
                           "best_us": cdr.best_lat, "start_us": cdr.records[0][1],
                           "wall_s": time.perf_counter() - t1}
        prof_line = {"config": args.profile_config, "candidates": args.n_cand, "warmup": 2, "iters": 10,
                     "knobs": {"sm_partition_rule": pknobs[0], "claim_depth": pknobs[1],
                               "steal": pknobs[2] if len(pknobs) > 2 else 2},
                     "schedules_per_s": args.n_cand / dt, "wall_s": dt,
                     "feasible": int((st_p == 0).sum()),
                     "best_us": float(np.nanmin(lat_p)) if len(lat_p) else None,
                     "median_us": float(np.nanmedian(lat_p)) if len(lat_p) else None,
                     "gather": "NCCL all_gather of per-rank latencies" if ws > 1 else "none (1 GPU)",
                     "rank_scales": pinfo.get("scales"),
                     "search": search_line}

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu:
        cms, reps, cores = oracle_sample(args.config)
        cpu = {"value": cms, "unit": "ms", "cores": cores, "kind": "oracle",
               "sample": f"{reps} full multi-tenant forward passes of {args.config} (all tenants, one batch), "
                         f"numpy fp64 with bf16 storage emulation"}

    if rank == 0:
        best_seq = min(base.get("seq", 1e9), base.get("seq_graph", 1e9))
        best_ms = min(base.get(m, 1e9) for m in ("ms_dfs", "ms_bfs", "ms_graph")) if base else 1e9
        line = {
            "metric": METRIC, "value": ms, "unit": "ms", "n_gpus": ws, "steps": K, "warmup": W,
            "ms_per_step": ms, "higher_is_better": False, "scaling": "weak", "vs_baseline": None,
            "latency_stats_ms": {"mean": float(np.mean(step_ms)), "median": float(np.median(step_ms)),
                                 "p90": float(np.percentile(step_ms, 90)), "rank": rank},
            "dtype": "bf16", "data": "synthetic (seeded LeCun-normal weights, identity-BN, N(0,1) input)",
            "config": {"workload": f"{args.config} ({CONFIG_NAMES.get(args.config, args.config)}): "
                                   + configs.CONFIGS[args.config][3],
                       "schedule": head_name, "stages": n_stages,
                       "sm_partition_rule": {0: "roofline-proportional", 1: "latency-balanced",
                                             2: "work/span"}[knobs[0]],
                       "claim_depth": knobs[1], "steal": knobs[2] if len(knobs) > 2 else 2,
                       "l2": "warm" if args.warm_l2 else "flushed before every timed step (256 MiB write)",
                       "parallelism": f"replicas x{ws}" if ws > 1 else "1 GPU"},
            "gpu_launches": K,
            "e2e": {"value": e2e_ms, "unit": "ms", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
            "roofline": roof,
            "cpu_baseline": cpu,
            "schedules_ms": results,
            "stage_us": [round(s, 2) for s in stage_us],
            "baselines_ms": base,
            "speedup_vs_sequential": (best_seq / ms) if base else None,
            "speedup_vs_multistream": (best_ms / ms) if base else None,
            "profiling": prof_line,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
