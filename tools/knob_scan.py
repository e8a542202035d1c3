"""Median device makespan of every executor knob triple (partition rule, claim depth, steal) of
TenantMix.KNOBS for one mix, all-concurrent schedule -- the spectrum calibrate() chooses from.

  python tools/knob_scan.py --config c4 [--runs 9]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2111_14255_b200.session import TenantMix  # noqa: E402
from workloads import configs, zoo  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c4")
ap.add_argument("--runs", type=int, default=9)
a = ap.parse_args()
g = configs.tenants(a.config)
m = TenantMix(g)
m.set_input(zoo.make_input(g[0]))
best, med = m.calibrate(runs=a.runs)
for k, v in sorted(med.items(), key=lambda kv: kv[1]):
    print(f"{a.config} knobs {k}: {v:.1f} us{'  <- chosen' if k == best else ''}")
