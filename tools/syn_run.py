"""Run a synthetic chain (see trace_exec --synthetic) through the executor, for ncu."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2111_14255_b200.session import TenantMix  # noqa: E402
from workloads import zoo  # noqa: E402

spec = sys.argv[1] if len(sys.argv) > 1 else "pw:960:960:7"
_, ci, co, hw = spec.split(":")
ci, co, hw = int(ci), int(co), int(hw)
b = zoo.GraphBuilder("tinyA", 1, ci, hw, hw, zoo.PREC_BF16, seed=0)
x = b.conv(-1, ci, 1, 1, 0)
for i in range(6):
    x = b.conv(x, co, 1, 1, 0)
    x = b.conv(x, ci, 1, 1, 0)
b.gap(x)
m = TenantMix([b.build()])
m.set_input(zoo.make_input(b.g))
m.ctx.set_schedule_pointers([[]])
for _ in range(4):
    m.run()
torch.cuda.synchronize()
