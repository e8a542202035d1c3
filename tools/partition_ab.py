"""Same-box A/B of the SM-partition rules (MT_OPT_PARTITION 0 = roofline-proportional,
1 = latency-balanced) and stealing modes on the executor: median makespan per config and schedule.

  python tools/partition_ab.py --configs c2,c3,c4 --runs 30 [--steal 2]
"""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2111_14255_b200 import mt  # noqa: E402
from paper_2111_14255_b200.session import TenantMix  # noqa: E402
from workloads import configs, zoo  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--configs", default="c2,c3,c4")
ap.add_argument("--runs", type=int, default=30)
ap.add_argument("--modes", default="0:2,1:2", help="partition:steal[:claim_depth] tuples")
ap.add_argument("--out", default=None)
a = ap.parse_args()
modes = [tuple(int(v) for v in m.split(":")) for m in a.modes.split(",")]
res = {}
for cfg in a.configs.split(","):
    g = configs.tenants(cfg)
    m = TenantMix(g)
    m.set_input(zoo.make_input(g[0]))
    L = [x.n_ops for x in g]
    scheds = {"all_concurrent": configs.all_concurrent_pointers(L), "uniform4": configs.uniform_pointers(L),
              "sequential": configs.sequential_pointers(L)}
    for sname, rho in scheds.items():
        m.ctx.set_schedule_pointers(rho)
        ts = {md: [] for md in modes}
        for rep in range(a.runs):
            for md in (modes if rep % 2 == 0 else modes[::-1]):
                m.ctx.set_option(mt.MT_OPT_PARTITION, md[0])
                m.ctx.set_option(mt.MT_OPT_STEAL, md[1])
                m.ctx.set_option(mt.MT_OPT_CLAIM_DEPTH, md[2] if len(md) > 2 else 0)
                if rep == 0:
                    for _ in range(3):
                        m.run()
                ts[md].append(m.run()[0])
        row = {"p%ds%d" % md[:2] + ("d%d" % md[2] if len(md) > 2 else ""): round(statistics.median(v), 1)
               for md, v in ts.items()}
        m.ctx.set_option(mt.MT_OPT_CLAIM_DEPTH, 0)
        m.ctx.set_option(mt.MT_OPT_PARTITION, 1)
        row["sms_balanced"] = m.ctx.sm_partition().tolist()
        m.ctx.set_option(mt.MT_OPT_PARTITION, 0)
        row["sms_roofline"] = m.ctx.sm_partition().tolist()
        res[f"{cfg}/{sname}"] = row
        print(cfg, sname, row, flush=True)
    del m
if a.out:
    json.dump(res, open(a.out, "w"), indent=1)
