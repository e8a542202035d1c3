"""SURVEY §8(f) f3 (first half): the paper's DFS vs BFS operator-invoking stall (P:481-494,
fig:bfs: 102.75 -> 51.23 us and 177.27 -> 51.23 us) re-measured on B200 with the host-launched
multi-stream baselines (one stream per tenant, the same tile kernels), next to the persistent
executor that has no host issue at all.  Stall of tenant i = device time of its first tile's
start minus the first tile start of the run (device trace, %globaltimer).

  python tools/issue_stall.py --config c3 --runs 5 [--out gpurun_out/issue_stall.json]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2111_14255_b200.session import TenantMix  # noqa: E402
from workloads import configs, zoo  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c3")
ap.add_argument("--runs", type=int, default=5)
ap.add_argument("--out", default="gpurun_out/issue_stall.json")
a = ap.parse_args()
g = configs.tenants(a.config)
L = [x.n_ops for x in g]
base = np.cumsum([0] + L)
m = TenantMix(g)
m.set_input(zoo.make_input(g[0]))
m.ctx.set_schedule_pointers(configs.all_concurrent_pointers(L))
cap = 1 << 20
buf = torch.zeros(cap * 16, dtype=torch.int64, device="cuda")


def traced(fn):
    m.ctx.set_trace(buf.data_ptr(), cap)
    fn()
    torch.cuda.synchronize()
    n = min(m.ctx.trace_count(), cap)
    t = buf[: n * 16].view(n, 16).cpu().numpy()
    m.ctx.set_trace(0, 0)
    return t


res = {"config": a.config, "tenants": [x.name for x in g], "ops": L}
for mode in ("ms_dfs", "ms_bfs", "executor"):
    stalls, spans, last_start = [], [], []
    for _ in range(a.runs + 1):
        box = {}
        fn = (lambda: box.setdefault("us", m.run()[0])) if mode == "executor" else \
            (lambda: box.setdefault("us", m.ctx.run_baseline(mode, m.in_ptrs, m.out_ptrs)))
        t = traced(fn)
        op = (t[:, 0] & 0xffffffff).astype(np.int64)
        ten = np.searchsorted(base, op, side="right") - 1
        t0 = t[:, 2].min()
        stalls.append([(t[ten == i, 2].min() - t0) / 1e3 for i in range(len(L))])
        # when each tenant's LAST op started: the accumulated issue delay the paper's DFS adds
        last_start.append([(t[op == base[i] + L[i] - 1, 2].min() - t0) / 1e3 for i in range(len(L))])
        spans.append(box["us"])
    stalls, last_start = np.array(stalls[1:]), np.array(last_start[1:])
    res[mode] = {"first_op_stall_us": np.median(stalls, 0).round(2).tolist(),
                 "last_op_start_us": np.median(last_start, 0).round(2).tolist(),
                 "makespan_us": float(np.median(spans[1:]))}
    print(mode, json.dumps(res[mode]), flush=True)
os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
json.dump(res, open(a.out, "w"), indent=1)
