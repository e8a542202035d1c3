"""Where the bench step's time goes outside the stages: CUDA-event time of one executor launch
vs its device stamps (first stamp after the co-residency barrier -> last barrier) vs the stage
time, L2 flushed before every run as in bench.py.

  python tools/overhead_probe.py --config c2 --knobs 1,3
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2111_14255_b200.session import TenantMix  # noqa: E402
from workloads import configs, zoo  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--knobs", default="1,3")
ap.add_argument("--runs", type=int, default=30)
a = ap.parse_args()
g = configs.tenants(a.config)
m = TenantMix(g)
m.set_input(zoo.make_input(g[0]))
m.ctx.set_schedule_pointers(configs.all_concurrent_pointers([x.n_ops for x in g]))
m.set_knobs(tuple(int(v) for v in a.knobs.split(",")))
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
st = torch.cuda.current_stream()
for _ in range(5):
    m.run()
ev, tot, stg = [], [], []
for i in range(a.runs):
    flush.fill_(1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    m.ctx.run_async(m.in_ptrs, m.out_ptrs, st.cuda_stream)
    e1.record(st)
    torch.cuda.synchronize()
    ev.append(e0.elapsed_time(e1) * 1e3)
    flush.fill_(1)
    torch.cuda.synchronize()
    t, s = m.run(st.cuda_stream)
    tot.append(t)
    stg.append(sum(s))
print(f"{a.config}: event {np.median(ev):.1f} us | device makespan (stamps) {np.median(tot):.1f} us | "
      f"stages {np.median(stg):.1f} us | prologue (pack + barrier) {np.median(tot) - np.median(stg):.1f} us | "
      f"launch + co-residency barrier + teardown {np.median(ev) - np.median(tot):.1f} us")
