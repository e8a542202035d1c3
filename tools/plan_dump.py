"""Print how every op of a config is executed (mt_op_plan; host-only context, no GPU needed).

  python tools/plan_dump.py --config c2
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2111_14255_b200 import mt  # noqa: E402
from workloads import configs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
a = ap.parse_args()
g = configs.tenants(a.config)
c = mt.Context(-1)
c.load_graphs(g, [[(0x1000, 0x2000, 0x3000) if x.params[j] else None for j in range(x.n_ops)] for x in g])
for t, gr in enumerate(g):
    for j in range(gr.n_ops):
        p = c.op_plan(t, j)
        nd = gr.nodes[j]
        print(f"{gr.name}:{j:3d} k{nd['kind']}:{nd.get('kh',0)}x{nd.get('kw',0)} {str(gr.shapes[j]):18s} " +
              " ".join(f"{k}={v}" for k, v in p.items()))
