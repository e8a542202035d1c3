"""Run the executor (or a baseline) of one config a few times -- a short command for ncu.

  python tools/prof_exec.py --config c2 --schedule all_concurrent --runs 5 [--baseline seq]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2111_14255_b200.session import TenantMix  # noqa: E402
from workloads import configs, zoo  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--schedule", default="all_concurrent")
ap.add_argument("--runs", type=int, default=5)
ap.add_argument("--baseline", default=None)
ap.add_argument("--steal", type=int, default=2)
ap.add_argument("--knobs", default="0,0", help="partition rule, claim depth (TenantMix.calibrate)")
ap.add_argument("--stage-split", action="store_true", help="one executor launch per stage (ncu per stage)")
ap.add_argument("--cps", type=int, default=1, help="executor CTAs per SM (2: f4 co-residency build)")
a = ap.parse_args()
g = configs.tenants(a.config)
L = [x.n_ops for x in g]
m = TenantMix(g, steal=a.steal, ctas_per_sm=a.cps)
m.set_input(zoo.make_input(g[0]))
rho = {"all_concurrent": configs.all_concurrent_pointers, "sequential": configs.sequential_pointers,
       "uniform4": configs.uniform_pointers}[a.schedule](L)
m.ctx.set_schedule_pointers(rho)
m.set_knobs(tuple(int(v) for v in a.knobs.split(",")))
if a.stage_split:
    m.ctx.set_option(7, 1)
for i in range(a.runs):
    if a.baseline:
        us = m.ctx.run_baseline(a.baseline, m.in_ptrs, m.out_ptrs)
        print(f"run {i}: baseline {a.baseline} {us:.1f} us")
    else:
        us, st = m.run()
        print(f"run {i}: {us:.1f} us, stages {[round(s, 1) for s in st]}")
torch.cuda.synchronize()
