"""Pins of the analytic pre-filter (oracle/costmodel.py) against SPEC.md cost_model's worked
examples and invariants and closed forms, then the C ABI (mt_estimate_batch_pointers,
host-only) against the oracle on real mixes and random candidates."""
import math
import random

import numpy as np
import pytest
from scipy import stats

from oracle import costmodel as cm
from oracle import ir
from workloads import configs

PRM = dict(peak_flops=1e12, mem_bw=1e9, op_latency_us=0.0, sync_us=0.0, c_compute=0.0, c_memory=0.0,
           max_concurrency=4)


def test_roofline_base_case():
    """S: 'one stream, one operator, flops=F, bytes=B, zero overheads -> max(F/peak, B/bw)'"""
    assert cm.estimate([[(3e6, 1e3)]], [[(0, 1)]], PRM) == pytest.approx(3.0)     # compute: 3 us
    assert cm.estimate([[(1e3, 5e3)]], [[(0, 1)]], PRM) == pytest.approx(5.0)     # memory: 5 us


def test_eq4_stage_longest_chain():
    """S: Eq.4 stage [S1(1,2,3), S2(1), S3(1,2)], unit ops, no contention -> 3 units"""
    costs = [[(0, 0)] * 10, [(0, 0)] * 4, [(0, 0)] * 5]
    prm = dict(PRM, op_latency_us=1.0)
    assert cm.estimate(costs, [[(0, 3), (0, 1), (0, 2)]], prm) == pytest.approx(3.0)


def test_two_compute_bound_ops_closed_form():
    """two identical compute-saturating ops in two streams of one stage: the device does 2F of
    work -> 2t; contention c adds 2t * c * (2-1)/max_concurrency; sequentially 2t as well"""
    t = 4.0
    costs = [[(t * 1e6, 0)], [(t * 1e6, 0)]]
    one = [[(0, 1), (0, 1)]]
    assert cm.estimate(costs, one, PRM) == pytest.approx(2 * t)
    assert cm.estimate(costs, one, dict(PRM, c_compute=0.6)) == pytest.approx(2 * t * (1 + 0.6 / 4))
    seq = ir.T([1, 1], configs.sequential_pointers([1, 1]))[1]
    assert cm.estimate(costs, seq, dict(PRM, sync_us=1.5)) == pytest.approx(2 * t + 2 * 1.5)


def _random_costs(L, rnd):
    return [[(rnd.uniform(0, 5e6), rnd.uniform(0, 5e3)) for _ in range(n)] for n in L]


def test_invariants_on_random_schedules():
    """S:241-247 invariants: (a) zero contention/overheads -> every valid schedule >= the longest
    stream's total, all-concurrent attains max(longest stream, total work); (b) c=0, sync>0:
    refining a schedule (splitting a stage) never lowers the estimate; (c) determinism"""
    rnd = random.Random(7)
    L = [3, 2, 3]     # 13,620 schedules
    costs = _random_costs(L, rnd)
    tot = [sum(max(F / 1e6, B / 1e3) for F, B in row) for row in costs]
    allc = ir.T(L, configs.all_concurrent_pointers(L))[1]
    Fc = sum(F for row in costs for F, B in row if F / 1e6 >= B / 1e3) / 1e6
    Mm = sum(B for row in costs for F, B in row if F / 1e6 < B / 1e3) / 1e3
    assert cm.estimate(costs, allc, PRM) == pytest.approx(max(max(tot), Fc, Mm))
    scheds = ir.enumerate_schedules(tuple(L))
    for s in rnd.sample(scheds, 300):
        assert cm.estimate(costs, s, PRM) >= max(tot) - 1e-9
        assert cm.estimate(costs, s, PRM) == cm.estimate(costs, s, PRM)
    prm = dict(PRM, sync_us=2.0)
    checked = 0
    for s in rnd.sample(scheds, 200):
        k = rnd.randrange(len(s))
        (stage, ) = [s[k]]
        # split stage k after its first non-empty tenant slice's first op
        cut = [(b, b + 1 if (e > b and i == next(q for q, (bb, ee) in enumerate(stage) if ee > bb)) else b)
               for i, (b, e) in enumerate(stage)]
        rest = [(c1, e) for (c0, c1), (b, e) in zip(cut, stage)]
        if all(c1 == c0 for c0, c1 in cut) or all(e == c1 for (c0, c1), (b, e) in zip(cut, stage)):
            continue
        finer = s[:k] + [cut, rest] + s[k + 1:]
        assert ir.validate(L, finer)[0] == ir.E_OK
        assert cm.estimate(costs, finer, prm) >= cm.estimate(costs, s, prm) + 2.0 - 1e-9
        checked += 1
    assert checked >= 50


def test_spearman_matches_scipy():
    rnd = random.Random(3)
    for _ in range(20):
        x = [rnd.choice([1, 2, 3, 4.5, 7]) for _ in range(30)]
        y = [rnd.random() for _ in range(30)]
        assert cm.spearman(x, y) == pytest.approx(stats.spearmanr(x, y)[0], abs=1e-12)


@pytest.mark.parametrize("config", ["c2", "c3", "c4"])
def test_abi_estimate_matches_oracle(config):
    mt = pytest.importorskip("paper_2111_14255_b200.mt")
    from .test_abi_host import host_ctx
    graphs = configs.tenants(config)
    L = [g.n_ops for g in graphs]
    c = host_ctx(graphs)
    costs = [[c.op_cost(t, j) for j in range(L[t])] for t in range(len(L))]
    cands = configs.sample_candidates(L, 200, seed=11)
    prm = dict(peak_flops=1.6e15, mem_bw=6.5e12, op_latency_us=4.5, sync_us=3.0, c_compute=0.3, c_memory=0.6,
               max_concurrency=4)
    est, st = c.estimate_batch_pointers(cands, **prm)
    for k, rho in enumerate(cands):
        status, ranges = ir.T(L, rho)
        if status[0] != ir.E_OK:
            assert st[k] == mt.MT_ERR_VALIDATION and math.isnan(est[k])
            continue
        assert st[k] == mt.MT_OK
        assert est[k] == pytest.approx(cm.estimate(costs, ranges, prm), rel=1e-12)
    assert np.isfinite(est[st == 0]).all()
