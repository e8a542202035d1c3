"""Synthetic single-tenant chains for profiling one tile kind (dwchain | pwchain | relu)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2111_14255_b200.session import TenantMix  # noqa: E402
from workloads import zoo  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--kind", default="dwchain")
ap.add_argument("--runs", type=int, default=3)
ap.add_argument("--baseline", default="seq")
a = ap.parse_args()
b = zoo.GraphBuilder("tinyA", 1, 384, 14, 14, zoo.PREC_BF16, seed=0)
x = b.conv(-1, 384, 1, 1, 0)
for i in range(6):
    x = b.conv(x, 384, 3, 1, 1, groups=384) if a.kind == "dwchain" else b.conv(x, 384, 1, 1, 0)
b.gap(x)
m = TenantMix([b.build()])
m.set_input(zoo.make_input(b.g))
m.ctx.set_schedule_pointers([[]])
for _ in range(a.runs):
    if a.baseline == "none":
        m.run()
    else:
        m.ctx.run_baseline(a.baseline, m.in_ptrs, m.out_ptrs)
torch.cuda.synchronize()
