"""Benchmark of the multi-tenant stage executor (BASELINE.json metric: multi-tenant latency ms vs
sequential / multi-stream; schedules profiled / sec).

One step = one mt_run of the whole hot path (input pack + every tenant op of every stage, one
cooperative launch) over one batch of the synthetic workload, inputs resident in HBM.
Default workload = BASELINE.json configs[3], the largest single-GPU configuration: the 5-tenant
mix ResNet-50 / Inception-v3 / VGG-16 / MobileNet-V2 / SqueezeNet 1.0 at 224x224, bf16.  `value`
is its batch-1 latency; the batch-8 leg of the same config is reported in the same line
(`batch8`).  configs[4] (1024 candidate schedules of the 3-tenant mix) is the `profiling` leg.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c4]

Multi-GPU (one process per GPU): with --gpus N > 1 and no WORLD_SIZE in the environment, bench.py
re-launches itself under torch.distributed.run with N ranks.  The executor runs as independent
replicas (a schedule's latency is a single-GPU property: DESIGN.md section 8, "replicas only");
the schedule-profiling leg shards candidates c -> rank c mod N with one NCCL all_gather of the
latencies, and Alg.1 coordinate descent gathers once per (round, row).
"""
from __future__ import annotations

import argparse
import json
import os
import socket
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
PROF_W, PROF_K = 2, 10          # profiling protocol (R8)


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c4")
    ap.add_argument("--b8-config", default="c4b8", help="second leg reported in the same line ('' = none)")
    ap.add_argument("--profile-config", default="c3")
    ap.add_argument("--n-cand", type=int, default=1024)
    ap.add_argument("--search-cand", type=int, default=64)
    ap.add_argument("--no-profile", action="store_true")
    ap.add_argument("--no-baselines", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--warm-l2", action="store_true", help="do not flush L2 between timed steps")
    return ap.parse_args(argv)


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def torchrun_cmd(n, argv, port):
    """the driver's own launch line for N ranks (one process per GPU, rendezvous on 127.0.0.1)"""
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
            "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *argv]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


def host_info():
    model = None
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                model = ln.split(":", 1)[1].strip()
                break
    except Exception:
        pass
    return {"cpu_model": model, "nproc": os.cpu_count()}


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
# CPU oracle timing (the only places bench.py executes oracle/): cpu_baseline and --impl reference
# ------------------------------------------------------------------------------------------
def _blas_threads():
    try:
        from threadpoolctl import threadpool_info
        return max((i.get("num_threads", 1) for i in threadpool_info()), default=1)
    except Exception:
        return os.cpu_count()


def oracle_pass_ms(config, reps_max, budget_s, threads=None):
    """mean wall time of full multi-tenant oracle forward passes (all tenants, one batch)"""
    from contextlib import nullcontext

    from oracle import forward as fw
    try:
        from threadpoolctl import threadpool_limits
        lim = threadpool_limits(threads) if threads else nullcontext()
    except Exception:
        lim = nullcontext()
    graphs = configs.tenants(config)
    x = zoo.make_input(graphs[0])
    times = []
    with lim:
        used = _blas_threads()
        t0 = time.perf_counter()
        while len(times) < reps_max and (not times or time.perf_counter() - t0 < budget_s):
            t1 = time.perf_counter()
            for g in graphs:
                fw.forward(g, x, "bf16")
            times.append(time.perf_counter() - t1)
    return float(np.mean(times)) * 1e3, len(times), used


def cpu_baseline(config):
    """The oracle as it stands, on this box's host cores: all BLAS threads and 1 thread."""
    ms_all, reps_all, cores = oracle_pass_ms(config, 3, 12.0)
    ms_one, reps_one, _ = oracle_pass_ms(config, 1, 0.0, threads=1)
    return {"value": ms_all, "unit": "ms", "cores": cores, "kind": "oracle",
            "sample": f"{reps_all} full multi-tenant forward passes of {config} (all tenants, one batch; "
                      f"numpy fp64 with bf16 storage emulation) on {cores} BLAS threads; "
                      f"{reps_one} pass on 1 thread",
            "value_1thread": ms_one, **host_info()}


def run_reference(args, ws, rank, budget_s=150.0):
    """The tier's reference arm: the CPU oracle as it stands, on the host cores.  A step = one
    full multi-tenant forward pass of the workload (all tenants, one batch).  At most one
    untimed warm-up pass (a pass of configs[3] takes seconds); timed passes stop at K or when the
    next would exceed budget_s (steps = passes done)."""
    if rank != 0:
        return
    cfg = args.config
    from oracle import forward as fw
    graphs = configs.tenants(cfg)
    x = zoo.make_input(graphs[0])

    def step():
        for g in graphs:
            fw.forward(g, x, "bf16")

    warm = min(args.warmup, 1)
    for _ in range(warm):
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
    cores = _blas_threads()
    line = {"impl": "reference", "metric": METRIC, "value": ms, "unit": "ms", "n_gpus": args.gpus,
            "steps": reps, "warmup": warm, "ms_per_step": ms, "higher_is_better": False,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{cfg} ({CONFIG_NAMES.get(cfg, cfg)}): " + configs.CONFIGS[cfg][3],
                       "parallelism": "cpu"},
            "cpu_baseline": {"value": ms, "unit": "ms", "cores": cores, "kind": "oracle",
                             "sample": f"{reps} full multi-tenant forward passes (all tenants, batch "
                                       f"{configs.CONFIGS[cfg][1]}), numpy fp64 with bf16 storage emulation",
                             **host_info()},
            "e2e": {"value": ms, "unit": "ms", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------------------
# rooflines: per stage max(F_s / TC, B_s / HBM), B_s = B_min of the stage
# ------------------------------------------------------------------------------------------
def op_tables(ctx, graphs):
    """per op: F (2*MACs, from the library's op cost) and weight bytes (bf16 conv/FC weights)"""
    F, Wb = [], []
    for t, g in enumerate(graphs):
        F.append([ctx.op_cost(t, j)[0] for j in range(g.n_ops)])
        Wb.append([2 * int(np.prod(p["weight"].shape)) if p and "weight" in p else 0 for p in g.params])
    return F, Wb


def stage_rooflines(ranges, graphs, F, Wb, tc_flops, hbm_bps, in_bytes):
    """per-stage roofline seconds.  B_min of a stage = weights of its ops + the shared input if a
    tenant starts there (read once) + fp32 logits of the tenants that end there."""
    out = []
    for st in ranges:
        f = b = 0
        starts = False
        for t, (lo, hi) in enumerate(st):
            f += sum(F[t][lo:hi])
            b += sum(Wb[t][lo:hi])
            starts |= lo == 0 and hi > 0
            if hi == graphs[t].n_ops and hi > lo:
                b += graphs[t].batch * graphs[t].out_classes * 4
        b += in_bytes if starts else 0
        out.append((max(f / tc_flops, b / hbm_bps), f, b))
    return out


# ------------------------------------------------------------------------------------------
# profiling leg (configs[4]): sharded profiling + Alg.1 over P, host plumbing only (tested on
# gloo with a stand-in profiler in tests/test_distributed_gloo.py)
# ------------------------------------------------------------------------------------------
def profiling_leg(pfn, cands, lengths, rank, ws, device=None, cd=True, cd_p=(0, 1, 2, 3), cd_m=8):
    from paper_2111_14255_b200 import distributed as D
    from paper_2111_14255_b200 import search as S
    info = {}
    t0 = time.perf_counter()
    lat, st = D.profile_distributed(pfn, cands, rank, ws, device=device,
                                    ref=(0, 1) if ws > 1 else None, info=info)
    wall = time.perf_counter() - t0
    out = {"lat": lat, "st": st, "wall_s": wall, "rank_scales": info.get("scales")}
    if cd:
        dpfn = (lambda cs: D.profile_distributed(pfn, cs, rank, ws, device=device)) if ws > 1 else pfn
        t1 = time.perf_counter()
        r = S.coordinate_descent_over_p(dpfn, lengths, cd_p, rounds=1, m=cd_m, seed=14255)
        out["cd"] = {"algorithm": f"coordinate descent (Alg.1) over P in {list(cd_p)}, R=1, M={cd_m}, "
                                  f"candidates sharded over {ws} rank(s), one all_gather per (round, row)",
                     "evaluations": r.evaluations, "best_us": r.best_lat, "best_P": len(r.best_rho[0]),
                     "wall_s": time.perf_counter() - t1}
    return out


# ------------------------------------------------------------------------------------------
# our arm
# ------------------------------------------------------------------------------------------
def main(argv=None):
    args = parse(argv)
    ws, rank, local = dist_env()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        raise SystemExit(subprocess.call(torchrun_cmd(args.gpus, sys.argv[1:] if argv is None else argv,
                                                      _free_port())))
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
    pk = peaks()
    hbm = pk.get("hbm_gbs", 6650.0)
    tc = pk.get("bf16_tflops", 1590.0)

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
        """measured executor knobs (partition rule, claim depth, steal); every rank uses rank 0's
        choice so latencies stay comparable across ranks"""
        kn, med = m.calibrate()
        if ws > 1:
            t = torch.tensor(list(kn), dtype=torch.int64, device=dev)
            dist.broadcast(t, 0)
            kn = tuple(int(v) for v in t.tolist())
            m.set_knobs(kn)
        return kn

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

    def leg(cfg, steps, search_cand, clk=None, headline=False):
        """one config: knob calibration + schedule search (untimed), then the timed steps of the best
        schedule, its per-stage rooflines, and the per-op-launch baselines of the same kernels"""
        graphs = configs.tenants(cfg)
        L = [g.n_ops for g in graphs]
        x = zoo.make_input(graphs[0])
        # executor configuration by measurement (like the knobs): 1 CTA per SM, or f4's two
        # co-resident CTAs per SM (MT_OPT_CTAS_PER_SM; bit-identical outputs) -- each calibrated,
        # the faster kept (rank 0 decides for every rank)
        cal = {}
        for cps in (1, 2):
            try:
                m = TenantMix(graphs, device=local, ctas_per_sm=cps)
            except Exception:   # e.g. fp32 tenants: 1 CTA/SM only
                continue
            m.set_input(x)
            kn, med = m.calibrate()
            cal[cps] = (m, kn, med[kn])
        cps = min(cal, key=lambda c: cal[c][2])
        if ws > 1:
            t = torch.tensor([cps], dtype=torch.int64, device=dev)
            dist.broadcast(t, 0)
            cps = int(t.item())
        mix = cal[cps][0]
        cal_us = {c: round(v[2], 2) for c, v in cal.items()}
        cal.clear()
        ctx = mix.ctx
        knobs = same_knobs(mix)
        cands = configs.sample_candidates(L, search_cand, seed=14255)
        named = {"all_concurrent": configs.all_concurrent_pointers(L),
                 "sequential": configs.sequential_pointers(L),
                 "uniform4": configs.uniform_pointers(L)}
        lat, st = ctx.profile_batch_pointers(cands, mix.in_ptrs, mix.out_ptrs, warmup=2, iters=5, stream=sp)
        named["best_of_%d" % len(cands)] = cands[int(np.nanargmin(np.where(st == 0, lat, np.nan)))]
        sched_ms = {}
        for name, rho in named.items():
            ctx.set_schedule_pointers(rho)
            sched_ms[name] = maxall(float(np.mean(time_steps(
                lambda: ctx.run_async(mix.in_ptrs, mix.out_ptrs, sp), max(steps // 4, 20), W))))
        head = min(sched_ms, key=sched_ms.get)
        ctx.set_schedule_pointers(named[head])
        if clk is not None:   # bring clocks under load before the headline timing
            t_end = time.time() + 0.4
            while time.time() < t_end:
                ctx.run_async(mix.in_ptrs, mix.out_ptrs, sp)
        step_ms = time_steps(lambda: ctx.run_async(mix.in_ptrs, mix.out_ptrs, sp), steps, W)
        ms = maxall(float(np.mean(step_ms)))
        _, stage_us = ctx.run(mix.in_ptrs, mix.out_ptrs, sp)
        # rooflines: the whole mix (one stage) and per stage of the timed schedule
        F, Wb = op_tables(ctx, graphs)
        ranges = np.asarray(ctx.get_schedule()).reshape(-1, len(L), 2).tolist()
        mix_roof = stage_rooflines([[[0, l] for l in L]], graphs, F, Wb, tc * 1e12, hbm * 1e9, x.nbytes)[0]
        st_roof = stage_rooflines(ranges, graphs, F, Wb, tc * 1e12, hbm * 1e9, x.nbytes)
        r = {"workload": f"{cfg} ({CONFIG_NAMES.get(cfg, cfg)}): " + configs.CONFIGS[cfg][3],
             "ms": ms, "schedule": head, "stages": len(ranges),
             "knobs": {"sm_partition_rule": {0: "roofline-proportional", 1: "latency-balanced",
                                             2: "work/span"}[knobs[0]],
                       "claim_depth": knobs[1], "steal": knobs[2] if len(knobs) > 2 else 2,
                       "ctas_per_sm": cps, "calibration_us_by_ctas_per_sm": cal_us},
             "latency_stats_ms": {"mean": float(np.mean(step_ms)), "median": float(np.median(step_ms)),
                                  "p90": float(np.percentile(step_ms, 90)), "rank": rank},
             "schedules_ms": sched_ms, "stage_us": [round(s, 2) for s in stage_us],
             "flops": int(mix_roof[1]), "bytes_min": int(mix_roof[2]),
             "stage_roofline": [{"us": round(s[0] * 1e6, 3), "bound": "tensor" if s[1] / (tc * 1e12) >= s[2] / (hbm * 1e9)
                                 else "hbm", "frac": round(s[0] * 1e6 / max(u, 1e-9), 4)}
                                for s, u in zip(st_roof, stage_us)],
             "schedule_roofline_us": round(sum(s[0] for s in st_roof) * 1e6, 3)}
        if not args.no_baselines:
            base = {}
            for mode in ("seq", "seq_graph", "ms_dfs", "ms_bfs", "ms_graph", "stage_events"):
                base[mode] = maxall(float(np.mean(time_steps(
                    lambda: ctx.run_baseline(mode, mix.in_ptrs, mix.out_ptrs, sp), max(steps // 4, 20), W))))
            # SEQ with single-tenant plans: each tenant alone in its own context (tile plans sized
            # for the whole GPU, not the mix's share), run back to back = sequential execution
            seq1 = {"seq": 0.0, "seq_graph": 0.0}
            for g in graphs:
                solo = TenantMix([g], device=local)
                solo.set_input(x)
                for mode in seq1:
                    seq1[mode] += maxall(float(np.mean(time_steps(
                        lambda: solo.ctx.run_baseline(mode, solo.in_ptrs, solo.out_ptrs, sp),
                        max(steps // 8, 10), W))))
                del solo
            base["seq_single_tenant_plans"] = seq1["seq"]
            base["seq_graph_single_tenant_plans"] = seq1["seq_graph"]
            best_seq = min(base[m] for m in ("seq", "seq_graph", "seq_single_tenant_plans",
                                             "seq_graph_single_tenant_plans"))
            best_ms = min(base[m] for m in ("ms_dfs", "ms_bfs", "ms_graph", "stage_events"))
            r.update(baselines_ms=base, speedup_vs_sequential=best_seq / ms, speedup_vs_multistream=best_ms / ms)
        if headline:
            # end to end through the C ABI with HOST buffers (pinned): H2D + D2H in the timed region
            xh = torch.from_numpy(x).pin_memory()
            outs_h = [torch.empty(o.shape, dtype=torch.float32).pin_memory() for o in mix.outputs]
            e2e = [ctx.run_host([xh.data_ptr()] * len(L), [o.data_ptr() for o in outs_h], sp)
                   for _ in range(W + steps)][W:]
            r["e2e"] = {"value": maxall(float(np.mean(e2e)) / 1e3), "unit": "ms",
                        "h2d_bytes_per_step": int(x.nbytes),
                        "d2h_bytes_per_step": int(sum(o.numel() * 4 for o in outs_h))}
        del mix
        torch.cuda.empty_cache()
        return r

    with ClockSampler(local) as clk:
        b1 = leg(args.config, K, args.search_cand, clk=clk, headline=True)
        b8 = leg(args.b8_config, max(K // 2, 10), max(args.search_cand // 4, 8), clk=clk) if args.b8_config else None
    ms = b1["ms"]

    def roofline(r):
        """the dominant kernel (the executor: one launch = the whole step) against the bound of its
        mix: HBM with B_min algorithmic bytes, or the tensor pipe with F"""
        t_s = r["ms"] * 1e-3
        hbm_bound = r["bytes_min"] / (hbm * 1e9) >= r["flops"] / (tc * 1e12)
        traffic = None
        try:
            prof = json.load(open(os.path.join(ROOT, "profiles", "r02_executor_ncu.json")))
            key = r["workload"].split()[0] + ("_cr" if r["knobs"]["ctas_per_sm"] == 2 else "")
            traffic = prof.get(key, {}).get("dram_bytes_per_launch")
        except Exception:
            pass
        out = ({"bound": "hbm", "achieved": r["bytes_min"] / t_s / 1e9, "peak": hbm, "unit": "GB/s",
                "frac": r["bytes_min"] / t_s / 1e9 / hbm, "traffic": traffic, "algorithmic_bytes": r["bytes_min"]}
               if hbm_bound else
               {"bound": "tensor", "achieved": r["flops"] / t_s / 1e12, "peak": tc, "unit": "TFLOP/s",
                "frac": r["flops"] / t_s / 1e12 / tc, "traffic": traffic, "algorithmic_flops": r["flops"]})
        out["kernel"] = ("mtk_cr::executor_kernel (2 CTAs/SM, f4)" if r["knobs"]["ctas_per_sm"] == 2 else
                         "mtk::executor_kernel") + " (whole step = 1 launch)"
        out["peak_source"] = "MEASURED_PEAKS.json (burst)" if pk else "B200_PROFILING.md fallback"
        out["stage_fracs"] = [s["frac"] for s in r["stage_roofline"]]
        return out

    # ---- schedules profiled per second (configs[4]: 1024 candidates of the 3-tenant mix) ----
    prof_line = None
    if not args.no_profile:
        pg = configs.tenants(args.profile_config)
        pmix = TenantMix(pg, device=local)
        x = zoo.make_input(pg[0])
        pmix.set_input(x)
        PL = [g.n_ops for g in pg]
        allc = configs.sample_candidates(PL, args.n_cand, seed=14255)
        pknobs = same_knobs(pmix)
        pfn = lambda cs: pmix.ctx.profile_batch_pointers(cs, pmix.in_ptrs, pmix.out_ptrs, PROF_W, PROF_K, sp)
        pmix.ctx.profile_batch_pointers(allc[:8], pmix.in_ptrs, pmix.out_ptrs, 1, 1, sp)  # warm
        barrier()
        res = profiling_leg(pfn, allc, PL, rank, ws, device=dev)
        torch.cuda.synchronize(dev)
        dt = maxall(res["wall_s"])
        lat_all, st_all = res["lat"], res["st"]
        lat_p = lat_all[st_all == 0]
        # bound (SURVEY d.7): G * n / sum over feasible candidates of (W+K) * its schedule roofline
        F, Wb = op_tables(pmix.ctx, pg)
        roof_sum = 0.0
        for rho, s in zip(allc, st_all):
            if s != 0:
                continue
            pmix.ctx.set_schedule_pointers(rho)
            rg = np.asarray(pmix.ctx.get_schedule()).reshape(-1, len(PL), 2).tolist()
            roof_sum += sum(v[0] for v in stage_rooflines(rg, pg, F, Wb, tc * 1e12, hbm * 1e9, x.nbytes))
        bound = ws * args.n_cand / ((PROF_W + PROF_K) * roof_sum) if roof_sum > 0 else None
        sps = args.n_cand / dt
        prof_line = {"config": args.profile_config, "candidates": args.n_cand, "warmup": PROF_W, "iters": PROF_K,
                     "knobs": {"sm_partition_rule": pknobs[0], "claim_depth": pknobs[1],
                               "steal": pknobs[2] if len(pknobs) > 2 else 2},
                     "schedules_per_s": sps, "wall_s": dt,
                     "roofline_schedules_per_s": bound, "frac_of_roofline": (sps / bound) if bound else None,
                     "feasible": int((st_all == 0).sum()),
                     "best_us": float(np.nanmin(lat_p)) if len(lat_p) else None,
                     "median_us": float(np.nanmedian(lat_p)) if len(lat_p) else None,
                     "gather": "NCCL all_gather of per-rank latencies" if ws > 1 else "none (1 GPU)",
                     "rank_scales": res["rank_scales"], "search": res.get("cd")}
        del pmix
        torch.cuda.empty_cache()

    cpu = None
    if rank == 0 and not args.no_cpu:
        cpu = cpu_baseline(args.config)

    if rank == 0:
        line = {
            "metric": METRIC, "value": ms, "unit": "ms", "n_gpus": ws, "steps": K, "warmup": W,
            "ms_per_step": ms, "higher_is_better": False, "scaling": "weak", "vs_baseline": None,
            "latency_stats_ms": b1["latency_stats_ms"],
            "dtype": "bf16", "data": "synthetic (seeded LeCun-normal weights, identity-BN, N(0,1) input)",
            "config": {"workload": b1["workload"], "schedule": b1["schedule"], "stages": b1["stages"],
                       **b1["knobs"],
                       "l2": "warm" if args.warm_l2 else "flushed before every timed step (256 MiB write)",
                       "parallelism": f"replicas x{ws}" if ws > 1 else "1 GPU"},
            "gpu_launches": K,
            "replica_steps_per_s": ws * 1e3 / ms,
            "e2e": b1["e2e"],
            "roofline": roofline(b1),
            "cpu_baseline": cpu,
            "schedules_ms": b1["schedules_ms"],
            "stage_us": b1["stage_us"],
            "stage_roofline": b1["stage_roofline"],
            "schedule_roofline_us": b1["schedule_roofline_us"],
            "baselines_ms": b1.get("baselines_ms"),
            "speedup_vs_sequential": b1.get("speedup_vs_sequential"),
            "speedup_vs_multistream": b1.get("speedup_vs_multistream"),
            "batch8": None if b8 is None else {
                "workload": b8["workload"], "value": b8["ms"], "unit": "ms", "schedule": b8["schedule"],
                "stages": b8["stages"], "knobs": b8["knobs"], "latency_stats_ms": b8["latency_stats_ms"],
                "roofline": roofline(b8), "stage_us": b8["stage_us"], "stage_roofline": b8["stage_roofline"],
                "schedules_ms": b8["schedules_ms"], "baselines_ms": b8.get("baselines_ms"),
                "speedup_vs_sequential": b8.get("speedup_vs_sequential"),
                "speedup_vs_multistream": b8.get("speedup_vs_multistream")},
            "profiling": prof_line,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
