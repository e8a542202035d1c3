"""Micro-benchmark of one conv op through the baseline launcher (one op_kernel launch per run).

  python tools/op_bench.py --cin 512 --cout 512 --k 3 --s 1 --p 1 --hw 7 [--batch 1] [--runs 20]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2111_14255_b200.session import TenantMix  # noqa: E402
from workloads import zoo  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--cin", type=int, default=512)
ap.add_argument("--cout", type=int, default=512)
ap.add_argument("--k", type=int, default=3)
ap.add_argument("--s", type=int, default=1)
ap.add_argument("--p", type=int, default=1)
ap.add_argument("--hw", type=int, default=7)
ap.add_argument("--batch", type=int, default=1)
ap.add_argument("--groups", type=int, default=1)
ap.add_argument("--runs", type=int, default=20)
ap.add_argument("--internal", type=int, default=1)
ap.add_argument("--cps", type=int, default=1, help="executor CTAs per SM (2: f4 co-resident build)")
a = ap.parse_args()
b = zoo.GraphBuilder("tinyA", a.batch, a.cin, a.hw, a.hw, zoo.PREC_BF16, seed=0)
x = b.relu(-1) if a.internal else -1    # internal input: the conv takes the TMA operand path
x = b.conv(x, a.cout, a.k, a.s, a.p, groups=a.groups)
b.gap(x)
g = b.build()
m = TenantMix([g], ctas_per_sm=a.cps)
m.set_input(zoo.make_input(g))
m.ctx.set_schedule_pointers([[]])
ci = 1 if a.internal else 0
print("plan", m.ctx.op_plan(0, ci))
F = m.ctx.op_cost(0, ci)[0]
ts = []
for i in range(a.runs):
    ts.append(m.ctx.run_baseline("seq", m.in_ptrs, m.out_ptrs))
print(f"seq (pack+conv+gap) median {np.median(ts):.1f} us")
ts = [m.run()[0] for _ in range(a.runs)]
print(f"executor median {np.median(ts):.1f} us")
cap = 1 << 16
buf = torch.zeros(cap * 16, dtype=torch.int64, device="cuda")
m.ctx.set_trace(buf.data_ptr(), cap)
spans = []
for _ in range(5):
    m.run()
    n = min(m.ctx.trace_count(), cap)
    t = buf[: n * 16].view(n, 16).cpu().numpy()
    op = t[:, 0] & 0xffffffff
    r = t[op == ci]
    spans.append((r[:, 5].max() - r[:, 2].min()) / 1e3)
    m.ctx.set_trace(buf.data_ptr(), cap)
sp = float(np.median(spans))
print(f"conv op span (first pick -> last release) {sp:.1f} us: {F / sp / 1e6:.1f} TFLOP/s")

torch.cuda.synchronize()
