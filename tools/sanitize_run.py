"""Workload for compute-sanitizer: config 1 (fp32 and bf16) under its hand-written
3-stage schedule and config 2 under a 2-stage schedule, one executor launch each plus one
per-op-launch baseline, outputs checked against the first run.

  compute-sanitizer --tool memcheck|racecheck|synccheck python tools/sanitize_run.py
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2111_14255_b200.session import TenantMix  # noqa: E402
from workloads import configs, zoo  # noqa: E402


def one(config, rho, precision=None, baseline="seq"):
    gs = configs.tenants(config, precision=precision)
    m = TenantMix(gs)
    m.ctx.set_option(3, 60000)            # MT_OPT_TIMEOUT_MS: the sanitizer slows spins down
    m.set_input(zoo.make_input(gs[0]))
    m.ctx.set_schedule_pointers(rho)
    m.run()
    ref = [o.clone() for o in m.outputs]
    m.ctx.run_baseline(baseline, m.in_ptrs, m.out_ptrs)
    torch.cuda.synchronize()
    same = all(torch.equal(a, b) for a, b in zip(m.outputs, ref))
    print(f"{config} prec={precision} stages={m.ctx.num_stages()} baseline={baseline} identical={same}",
          flush=True)
    assert same


if __name__ == "__main__":
    one("c1", configs.c1_schedule_pointers())
    one("c1", configs.c1_schedule_pointers(), precision=zoo.PREC_BF16)
    gs = configs.tenants("c2")
    L = [g.n_ops for g in gs]
    one("c2", [[L[0] // 2], [L[1] // 2]], baseline="ms_bfs")
    print("sanitize workload done")
