"""Per-k-block mainloop rate of one tensor-core conv op (device trace stamps): for each tile, the
time from the first pipeline stage landing to the last MMA issue, divided by the k-blocks after the
first.  Distinguishes TMA-rate-bound mainloops from fixed per-tile costs.

  python tools/kb_rate.py --cin 960 --cout 160 --k 1 --hw 7 [--batch 1]
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
ap.add_argument("--cin", type=int, default=960)
ap.add_argument("--cout", type=int, default=160)
ap.add_argument("--k", type=int, default=1)
ap.add_argument("--hw", type=int, default=7)
ap.add_argument("--batch", type=int, default=1)
ap.add_argument("--flush", action="store_true", help="flush L2 before the traced run")
a = ap.parse_args()
b = zoo.GraphBuilder("tinyA", a.batch, a.cin, a.hw, a.hw, zoo.PREC_BF16, seed=0)
x = b.relu(-1)
x = b.conv(x, a.cout, a.k, 1, a.k // 2)
b.gap(x)
g = b.build()
m = TenantMix([g])
m.set_input(zoo.make_input(g))
m.ctx.set_schedule_pointers([[]])
plan = m.ctx.op_plan(0, 1)
for _ in range(3):
    m.run()
cap = 1 << 14
buf = torch.zeros(cap * 16, dtype=torch.int64, device="cuda")
fl = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
res = []
for rep in range(5):
    if a.flush:
        fl.fill_(1)
    m.ctx.set_trace(buf.data_ptr(), cap)
    m.run()
    n = m.ctx.trace_count()
    m.ctx.set_trace(0, 0)
    tr = buf[: n * 16].view(n, 16).cpu().numpy().astype(np.int64)
    r = tr[(tr[:, 0] & 0xffffffff) == 1]
    res.append(r)
r = np.concatenate(res)
nk = int(np.ceil(a.cin * a.k * a.k / 64 / max(plan["splits"], 1)))
first = (r[:, 8] - r[:, 3]) / 1e3
main = (r[:, 9] - r[:, 8]) / 1e3
epi = (r[:, 7] - r[:, 4]) / 1e3
iss0 = (r[:, 15] - r[:, 3]) / 1e3
issl = (r[:, 10] - r[:, 3]) / 1e3
print("plan", plan, "k-blocks per tile", nk)
print(f"deps->first stage {np.median(first):.2f} us; first->last MMA {np.median(main):.2f} us "
      f"({np.median(main) / max(nk - 1, 1) * 1e3:.0f} ns per k-block); acc->released {np.median(epi):.2f} us")
print(f"producer: first A issued {np.median(iss0):.2f} us, last A issued {np.median(issl):.2f} us after deps")
