"""the paper's own model-zoo mixes (Table I, Table II) on
one B200 -- the stage executor under the all-concurrent, sequential and searched schedules next
to the same kernels launched one per op (SEQ "CuDNN-Seq" analogue, multi-stream "Stream-Parallel"
analogue, the paper's stage/event mechanism).  Every number: CUDA events on the launching
stream, L2 flushed (256 MiB write) before every timed run, mean of --runs.

  python tools/zoo_table.py [--configs vgg_r18,r18_r34,...] [--runs 20] [--cands 128]
      [--out gpurun_out/zoo_table.json]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2111_14255_b200 import search as S  # noqa: E402
from paper_2111_14255_b200.session import TenantMix  # noqa: E402
from workloads import configs, zoo  # noqa: E402

TABLE = ["vgg_r18", "r18_r34", "r34_r50", "r50_r101", "vgg_r18_r50", "r18_r34_r50", "zoo5",
         "alex_vgg_r18", "r18_r34_r101", "r18_r50_r101"]
PAPER = {   # Table I (Titan V) / Table II (P6000): CuDNN-Seq, Stream-Parallel, Ours-C (ms) -- context
    "vgg_r18": ("I", 3.989, 3.638, 2.912), "r18_r34": ("I", 4.673, 3.743, 3.128),
    "r34_r50": ("I", 6.688, 5.449, 4.478), "r50_r101": ("I", 10.75, 8.588, 8.203),
    "vgg_r18_r50": ("I", 7.674, 6.522, 5.587), "r18_r34_r50": ("I", 8.344, 6.301, 5.096),
    "zoo5": ("I", 17.962, 12.848, 10.42), "alex_vgg_r18": ("II", 5.754, 4.694, 4.126),
    "r18_r34_r101": ("II", 14.278, 11.833, 10.463), "r18_r50_r101": ("II", 15.785, 12.32, 10.711),
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default=",".join(TABLE))
    ap.add_argument("--runs", type=int, default=20)
    ap.add_argument("--cands", type=int, default=128)
    ap.add_argument("--out", default="gpurun_out/zoo_table.json")
    ap.add_argument("--no-calibrate", action="store_true")
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    stream = torch.cuda.current_stream(dev)
    sp = stream.cuda_stream
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    def timed(fn, runs=a.runs, warm=3):
        for _ in range(warm):
            fn()
        torch.cuda.synchronize()
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(runs)]
        for e0, e1 in evs:
            flush.fill_(1)
            e0.record(stream)
            fn()
            e1.record(stream)
        torch.cuda.synchronize()
        return float(np.mean([e0.elapsed_time(e1) for e0, e1 in evs]))

    res = {}
    for cfg in a.configs.split(","):
        t0 = time.time()
        g = configs.tenants(cfg)
        L = [x.n_ops for x in g]
        r = {"tenants": list(configs.CONFIGS[cfg][0]), "ops": L}
        # executor configuration (1 or 2 CTAs per SM, f4) and knobs (partition rule, claim depth,
        # steal) chosen by measurement, as in bench.py
        cal = {}
        for cps in ((1, 2) if not a.no_calibrate else (1,)):
            try:
                mm = TenantMix(g, ctas_per_sm=cps)
            except Exception:
                continue
            mm.set_input(zoo.make_input(g[0]))
            if a.no_calibrate:
                cal[cps] = (mm, None, None, 0.0)
                continue
            kn, med = mm.calibrate()
            cal[cps] = (mm, kn, med, med[kn])
        cps = min(cal, key=lambda c: cal[c][3])
        m, kn, med, _ = cal[cps]
        r["ctas_per_sm"] = cps
        r["calibration_us_by_ctas_per_sm"] = {c: round(v[3], 1) for c, v in cal.items()}
        cal.clear()
        ctx = m.ctx
        run = lambda: ctx.run_async(m.in_ptrs, m.out_ptrs, sp)
        if kn is not None:
            r["knobs"] = {"sm_partition_rule": kn[0], "claim_depth": kn[1], "steal": kn[2] if len(kn) > 2 else 2,
                          "calibration_us": {",".join(map(str, k)): round(v, 1) for k, v in med.items()}}
        for name, rho in (("all_concurrent", configs.all_concurrent_pointers(L)),
                          ("sequential_schedule", configs.sequential_pointers(L)),
                          ("uniform4", configs.uniform_pointers(L))):
            ctx.set_schedule_pointers(rho)
            r[name] = timed(run)
        # random search (Ours-R analogue) and coordinate descent (Ours-C, Alg.1)
        pfn = lambda cs: ctx.profile_batch_pointers(cs, m.in_ptrs, m.out_ptrs, 2, 5, sp)
        rs = S.random_search(pfn, L, a.cands, seed=14255)
        ctx.set_schedule_pointers(rs.best_rho)
        r["random_search"] = {"candidates": a.cands, "best_rho": rs.best_rho, "profiled_us": rs.best_lat, "ms": timed(run)}
        cd = S.coordinate_descent(pfn, L, P=3, rounds=2, m=8, seed=14255)
        ctx.set_schedule_pointers(cd.best_rho)
        r["coordinate_descent"] = {"P": 3, "R": 2, "M": 8, "evaluations": cd.evaluations, "best_rho": cd.best_rho, "profiled_us": cd.best_lat,
                                   "ms": timed(run)}
        base = {}
        for mode in ("seq", "seq_graph", "ms_dfs", "ms_bfs", "ms_graph", "stage_events"):
            base[mode] = timed(lambda: ctx.run_baseline(mode, m.in_ptrs, m.out_ptrs, sp), max(a.runs // 2, 5))
        r["baselines"] = base
        best_exec = min(r["all_concurrent"], r["random_search"]["ms"], r["coordinate_descent"]["ms"])
        r["best_executor_ms"] = best_exec
        r["speedup_vs_seq"] = min(base["seq"], base["seq_graph"]) / best_exec
        r["speedup_vs_multistream"] = min(base["ms_dfs"], base["ms_bfs"], base["ms_graph"]) / best_exec
        if cfg in PAPER:
            r["paper_context"] = dict(zip(("table", "cudnn_seq_ms", "stream_parallel_ms", "ours_c_ms"), PAPER[cfg]))
        r["wall_s"] = time.time() - t0
        res[cfg] = r
        print(cfg, json.dumps({k: v for k, v in r.items() if k not in ("ops",)}), flush=True)
        del m, ctx
        torch.cuda.empty_cache()
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    json.dump(res, open(a.out, "w"), indent=1)
    open(a.out.replace(".json", ".md"), "w").write(render_md(res) + "\n")



def render_md(res):
    """Markdown table of a zoo_table JSON (profiles/<round>_zoo_table.md body)."""
    rows = ["| mix | CTAs/SM, knobs (rule, D, steal) | all-conc. | rand | coord (P3,R2,M8) | seq sched. | SEQ | SEQ_G | MS_BFS | MS_G "
            "| STAGE_EV | best vs SEQ_G | best vs MS_G | paper Seq / Stream / Ours-C |",
            "|---|---|---|---|---|---|---|---|---|---|---|---|---|---|"]
    for cfg, r in res.items():
        b = r["baselines"]
        kn = r.get("knobs")
        pc = r.get("paper_context")
        paper = f"{pc['cudnn_seq_ms']} / {pc['stream_parallel_ms']} / {pc['ours_c_ms']} ({pc['table']})" if pc else "-"
        rows.append(
            f"| {cfg}: {'+'.join(r['tenants'])} | {r.get('ctas_per_sm', 1)}, {(kn['sm_partition_rule'], kn['claim_depth'], kn.get('steal', 2)) if kn else '(0, 0, 2)'} "
            f"| {r['all_concurrent']:.3f} | {r['random_search']['ms']:.3f} | {r['coordinate_descent']['ms']:.3f} "
            f"| {r['sequential_schedule']:.3f} | {b['seq']:.3f} | {b['seq_graph']:.3f} | {b['ms_bfs']:.3f} "
            f"| {b['ms_graph']:.3f} | {b['stage_events']:.3f} | {min(b['seq'], b['seq_graph']) / r['best_executor_ms']:.2f}x "
            f"| {min(b['ms_dfs'], b['ms_bfs'], b['ms_graph']) / r['best_executor_ms']:.2f}x | {paper} |")
    return "\n".join(rows)


if __name__ == "__main__":
    main()
