"""Per-tile trace of one executor run (mt_set_trace): where does the time go?

  python tools/trace_exec.py --config c2 [--schedule all_concurrent] [--baseline seq] [--out f.json]
"""
import argparse
import collections
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2111_14255_b200.session import TenantMix  # noqa: E402
from workloads import configs, zoo  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--schedule", default="all_concurrent")
ap.add_argument("--baseline", default=None)
ap.add_argument("--out", default=None)
ap.add_argument("--top", type=int, default=30)
ap.add_argument("--partition", type=int, default=None)
ap.add_argument("--steal", type=int, default=None)
ap.add_argument("--claim", type=int, default=None)
ap.add_argument("--cps", type=int, default=1, help="executor CTAs per SM (2: f4 co-resident build)")
ap.add_argument("--synthetic", default=None, help="dwchain | pwchain | gapchain")
a = ap.parse_args()
if a.synthetic and a.synthetic.startswith("pw:"):
    # pw:CIN:COUT:HW  -> alternating 1x1 convs CIN->COUT->CIN at HWxHW
    _, ci, co, hw = a.synthetic.split(":")
    ci, co, hw = int(ci), int(co), int(hw)
    b = zoo.GraphBuilder("tinyA", 1, ci, hw, hw, zoo.PREC_BF16, seed=0)
    x = b.conv(-1, ci, 1, 1, 0)
    for i in range(6):
        x = b.conv(x, co, 1, 1, 0)
        x = b.conv(x, ci, 1, 1, 0)
    b.gap(x)
    g = [b.build()]
elif a.synthetic == "stempool":
    b = zoo.GraphBuilder("tinyA", 1, 3, 224, 224, zoo.PREC_BF16, seed=0)
    x = b.conv(-1, 64, 7, 2, 3)
    for i in range(4):
        x = b.maxpool(x, 3, 1, 1)
    x = b.maxpool(x, 3, 2, 1)
    b.gap(x)
    g = [b.build()]
elif a.synthetic:
    b = zoo.GraphBuilder("tinyA", 1, 384, 14, 14, zoo.PREC_BF16, seed=0)
    x = b.conv(-1, 384, 1, 1, 0)
    for i in range(12):
        if a.synthetic == "dwchain":
            x = b.conv(x, 384, 3, 1, 1, groups=384)
        elif a.synthetic == "pwchain":
            x = b.conv(x, 384, 1, 1, 0)
        else:
            x = b.relu(x)
    b.gap(x)
    g = [b.build()]
else:
    g = configs.tenants(a.config)
L = [x.n_ops for x in g]
m = TenantMix(g, ctas_per_sm=a.cps)
m.set_input(zoo.make_input(g[0]))
rho = {"all_concurrent": configs.all_concurrent_pointers, "sequential": configs.sequential_pointers,
       "uniform4": configs.uniform_pointers}[a.schedule](L)
m.ctx.set_schedule_pointers(rho)
if a.partition is not None:
    m.ctx.set_option(5, a.partition)
if a.steal is not None:
    m.ctx.set_option(1, a.steal)
if a.claim is not None:
    m.ctx.set_option(6, a.claim)
print("sm partition", m.ctx.sm_partition().tolist())
for _ in range(3):
    m.run()
cap = 1 << 16
buf = torch.zeros(cap * 16, dtype=torch.int64, device="cuda")
m.ctx.set_trace(buf.data_ptr(), cap)
if a.baseline:
    total = m.ctx.run_baseline(a.baseline, m.in_ptrs, m.out_ptrs)
    stages = []
else:
    total, stages = m.run()
n = m.ctx.trace_count()
m.ctx.set_trace(0, 0)
tr = buf[: n * 16].view(n, 16).cpu().numpy().astype(np.int64)
t0 = tr[:, 2].min()
names = []
for t, gg in enumerate(g):
    for j in range(gg.n_ops):
        nd = gg.nodes[j]
        names.append(f"{gg.name[:8]}:{j}:{zoo.KIND_NAMES[nd['kind']]}{'dw' if nd['groups'] > 1 else ''}"
                     f"{nd['kh']}x{nd['kw']}s{nd['sh']}->{gg.shapes[j]}")
per = collections.defaultdict(list)
for r in tr:
    per[int(r[0] & 0xffffffff)].append(r)
rows = []
for op, rs in per.items():
    rs = np.array(rs)
    wait = (rs[:, 3] - rs[:, 2]) / 1e3
    work = (rs[:, 5] - rs[:, 3]) / 1e3
    mma = np.where(rs[:, 4] > 0, (rs[:, 4] - rs[:, 3]) / 1e3, 0)
    run = (rs[:, 7] - rs[:, 3]) / 1e3
    rel = (rs[:, 5] - rs[:, 7]) / 1e3
    span = (rs[:, 5].max() - rs[:, 2].min()) / 1e3
    rows.append(dict(op=op, name=names[op], tiles=len(rs), start=(rs[:, 2].min() - t0) / 1e3,
                     end=(rs[:, 5].max() - t0) / 1e3, span=span, wait_mean=wait.mean(), wait_max=wait.max(),
                     work_mean=work.mean(), work_max=work.max(), mma_mean=mma.mean(),
                     run_mean=run.mean(), rel_mean=rel.mean()))
rows.sort(key=lambda r: r["start"])
print(f"total {total:.1f} us, stages {[round(s, 1) for s in stages]}, tiles traced {n}")
print(f"{'op':>4} {'name':46} {'tiles':>5} {'start':>7} {'end':>7} {'wait':>6} {'work':>6} {'wmax':>6} {'mma':>6} {'run':>6} {'rel':>6}")
for r in rows:
    print(f"{r['op']:4d} {r['name'][:46]:46} {r['tiles']:5d} {r['start']:7.1f} {r['end']:7.1f} {r['wait_mean']:6.2f} "
          f"{r['work_mean']:6.2f} {r['work_max']:6.2f} {r['mma_mean']:6.2f} {r['run_mean']:6.2f} {r['rel_mean']:6.2f}")
# per-tenant SM occupancy (north star: "SM occupancy per tenant slice"): busy SM-us of the
# tenant's tiles, how many of them ran on CTAs homed on another tenant (stealing), and the busy
# fraction of the tenant's home CTAs over the makespan
bounds = np.cumsum([0] + L)
ten_of = np.searchsorted(bounds, (tr[:, 0] & 0xffffffff), side="right") - 1
home = tr[:, 6]
sms = m.ctx.sm_partition().tolist()
occ = []
for t in range(len(L)):
    sel = ten_of == t
    w = (tr[sel, 5] - tr[sel, 3]).sum() / 1e3
    stolen = int((home[sel] != t).sum())
    hsel = home == t
    hb = (tr[hsel, 5] - tr[hsel, 3]).sum() / 1e3
    n_home = sms[0][t] if len(sms) == 1 else None
    occ.append(dict(tenant=g[t].name, tiles=int(sel.sum()), busy_sm_us=round(float(w), 1), stolen_tiles=stolen,
                    home_ctas=n_home,
                    home_busy_frac=round(float(hb / (n_home * total)), 3) if n_home else None))
    print(f"tenant {g[t].name:14s} tiles {int(sel.sum()):5d} busy {w:8.1f} SM-us  run by other tenants' CTAs {stolen:5d}"
          + (f"  home CTAs {n_home:3d} busy {hb / (n_home * total):.3f} of makespan" if n_home else ""))
# per-CTA time split: waiting for dependencies (claimed, not ready), working (deps -> released),
# and between tiles (release -> next pick: claiming, retries of bounded claim-ahead, stage end)
cta = tr[:, 1] >> 32
wait_t = ((tr[:, 3] - tr[:, 2]).sum()) / 1e3
gap_t = 0.0
for c in np.unique(cta):
    r = tr[cta == c]
    r = r[np.argsort(r[:, 2])]
    gap_t += ((r[1:, 2] - r[:-1, 5]).clip(min=0).sum()) / 1e3
last_end = (tr[:, 5].max() - t0) / 1e3
print(f"CTA time: dependency wait {wait_t:.0f} us, between tiles {gap_t:.0f} us (summed over CTAs); "
      f"last release at {last_end:.1f} us of stage {stages[0] if stages else 0:.1f} us")
busy = ((tr[:, 5] - tr[:, 3]).sum() / 1e3)
print(f"SM-busy (work) us summed over CTAs: {busy:.1f}; makespan x CTAs: {total * 148:.1f} -> util {busy / (total * 148):.3f}")
if a.out:
    json.dump(dict(total=total, stages=stages, rows=rows, occupancy=occ), open(a.out, "w"), indent=1)
    np.save(a.out.replace(".json", "_raw.npy"), tr)
