"""Schedule executor oracle (TEST INFRASTRUCTURE ONLY).

Runs a validated stage schedule exactly as the paper describes its semantics:
  * stages in order; "all operators in the same stage must all finish so as to step into the
    next stage";
  * within a stage every tenant's slice, in operator order ("operators in one stream can only
    be launched sequentially"); tenants are independent and visited in index order;
  * before an operator runs, every operator it reads must already have run -- asserted, so a
    schedule that broke data-flow order would raise.
Its per-tenant outputs therefore equal the sequential forward pass, which is itself a test.
"""
from __future__ import annotations

import numpy as np

from . import ir
from .forward import eval_node, _round


def run_schedule(graphs, ranges, x_per_tenant, mode="exact"):
    st = ir.validate([g.n_ops for g in graphs], ranges)
    if st[0] != ir.E_OK:
        raise ValueError(f"invalid schedule {st}")
    acts = [dict() for _ in graphs]
    xin = [_round(np.asarray(x, dtype=np.float64), mode) for x in x_per_tenant]
    for stage in ranges:
        for t, (b, e) in enumerate(stage):
            g = graphs[t]
            for j in range(b, e):
                nd = g.nodes[j]
                deps = list(nd["inputs"]) + ([nd["residual"]] if nd["residual"] >= 0 else [])
                for d in deps:
                    assert d == -1 or d in acts[t], f"tenant {t} op {j} reads op {d} not yet run"
                ins = [xin[t] if i == -1 else acts[t][i] for i in nd["inputs"]]
                res = acts[t][nd["residual"]] if nd["residual"] >= 0 else None
                acts[t][j] = eval_node(nd, g.params[j], ins, res, mode, is_last=(j == g.n_ops - 1))
    return [acts[t][g.n_ops - 1].reshape(g.batch, -1) for t, g in enumerate(graphs)]
