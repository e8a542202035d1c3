"""heterogeneous co-residency (MT_OPT_CTAS_PER_SM = 2): two 128-thread executor
CTAs per SM (kernels_cr.cu), the SM's two slots serving a compute-bound and a memory-bound slice
(P:161-166).  Every op against the oracle; within the configuration, schedules change when tiles
run, never what they compute; against the 1-CTA executor the outputs agree within the
two runs' bf16 tolerances (its plans may split K differently).
Run: pytest -m gpu."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from workloads import configs, zoo  # noqa: E402

from .gpu_helpers import teacher_forced_errors  # noqa: E402

_MIXES = {}


def mix(config, cps):
    key = (config, cps)
    if key not in _MIXES:
        from paper_2111_14255_b200.session import TenantMix
        graphs = configs.tenants(config)
        m = TenantMix(graphs, ctas_per_sm=cps)
        x = zoo.make_input(graphs[0])
        m.set_input(x)
        m.x_np = x
        _MIXES[key] = m
    return _MIXES[key]


def _outs(m):
    torch.cuda.synchronize()
    return [o.clone() for o in m.outputs]


@pytest.mark.parametrize("config", ["c2", "c3", "c4", "c4b8"])
def test_coresident_teacher_forced_every_op(config):
    m = mix(config, 2)
    L = [g.n_ops for g in m.graphs]
    m.ctx.set_schedule_pointers(configs.all_concurrent_pointers(L))
    m.run()
    for t, g in enumerate(m.graphs):
        errs = teacher_forced_errors(m, m.x_np, t)
        worst = int(np.argmax(errs))
        assert max(errs) <= 1e-2, (g.name, worst, g.nodes[worst]["kind"], errs[worst])


@pytest.mark.parametrize("config", ["c2", "c4", "c4b8"])
def test_coresident_schedule_invariance_and_one_cta_agreement(config):
    """within the co-resident configuration, every schedule tried and the per-op-launch baselines
    of its build give the same bits (its plans size tiles for 2 x the CTAs, so split-K factors --
    and with them fp32 summation orders -- may differ from the 1-CTA plans: that comparison is
    within the bf16 tolerance instead)"""
    m1, m2 = mix(config, 1), mix(config, 2)
    L = [g.n_ops for g in m1.graphs]
    m1.ctx.set_schedule_pointers(configs.all_concurrent_pointers(L))
    m1.run()
    one = _outs(m1)
    m2.ctx.set_schedule_pointers(configs.all_concurrent_pointers(L))
    m2.run()
    ref = _outs(m2)
    for a, b in zip(ref, one):
        d = (a.double() - b.double()).abs().max().item()
        assert d <= 2e-2 * b.double().abs().max().item(), d   # both within 1e-2 of the oracle
    cands = [configs.all_concurrent_pointers(L), configs.sequential_pointers(L), configs.uniform_pointers(L)] + \
        configs.sample_candidates(L, 40, seed=11)[2:]
    n_ok = 0
    for rho in cands:
        try:
            m2.ctx.set_schedule_pointers(rho)
        except Exception:
            continue
        n_ok += 1
        for o in m2.outputs:
            o.fill_(float("nan"))
        m2.ctx.run_async(m2.in_ptrs, m2.out_ptrs)
        for a, b in zip(_outs(m2), ref):
            assert torch.equal(a, b), rho
    assert n_ok >= 30
    m2.ctx.set_schedule_pointers(configs.uniform_pointers(L))
    for mode in ("seq", "ms_bfs", "stage_events"):
        for o in m2.outputs:
            o.fill_(float("nan"))
        m2.ctx.run_baseline(mode, m2.in_ptrs, m2.out_ptrs)
        for a, b in zip(_outs(m2), ref):
            assert torch.equal(a, b), mode


def test_coresident_knobs_and_steal_off():
    """strict partition (no stealing: each tenant only on its own (slot, SM) homes) and the
    latency-balanced rule with bounded claim-ahead still complete with the same bits"""
    m2 = mix("c3", 2)
    L = [g.n_ops for g in m2.graphs]
    m2.ctx.set_schedule_pointers(configs.all_concurrent_pointers(L))
    m2.set_knobs((0, 0, 2))
    m2.run()
    ref = _outs(m2)
    m2.ctx.set_schedule_pointers(configs.uniform_pointers(L))
    for knobs in ((1, 2, 2), (0, 0, 0), (1, 0, 1)):
        m2.set_knobs(knobs)
        for o in m2.outputs:
            o.fill_(float("nan"))
        m2.run()
        for a, b in zip(_outs(m2), ref):
            assert torch.equal(a, b), knobs
    m2.set_knobs((0, 0, 2))


def test_coresident_profile_batch_and_host_run():
    """the profiling entry point (a10) and the host-buffer run in the co-resident configuration:
    statuses from the IR, finite latencies, and mt_run_host = the device run bit for bit"""
    from oracle import ir
    m = mix("c2", 2)
    L = [g.n_ops for g in m.graphs]
    cands = configs.sample_candidates(L, 16, seed=5)
    cands.append([[0, 0], [0, 0]])          # all-empty stages -> infeasible
    lat, st = m.ctx.profile_batch_pointers(cands, m.in_ptrs, m.out_ptrs, warmup=1, iters=3)
    for k, rho in enumerate(cands):
        ok = ir.T(L, rho)[0][0] == ir.E_OK
        assert (st[k] == 0) == ok
        assert (1.0 < lat[k] < 1e5) if ok else np.isnan(lat[k])
    m.ctx.set_schedule_pointers(configs.uniform_pointers(L))
    m.run()
    ref = _outs(m)
    xh = torch.from_numpy(m.x_np).pin_memory()
    outs_h = [torch.empty(o.shape, dtype=torch.float32).pin_memory() for o in m.outputs]
    m.ctx.run_host([xh.data_ptr()] * len(L), [o.data_ptr() for o in outs_h])
    for a, b in zip(outs_h, ref):
        assert torch.equal(a, b.cpu())


def test_coresident_stage_split_and_repeated_runs():
    """one launch per stage (the profiling mode) in the co-resident configuration: the (slot, SM)
    counters return to zero at every kernel exit, so every launch maps its CTAs again; outputs equal
    the single launch's, and 20 back-to-back runs stay bit-identical"""
    from paper_2111_14255_b200 import mt as M
    m = mix("c3", 2)
    L = [g.n_ops for g in m.graphs]
    m.ctx.set_schedule_pointers(configs.uniform_pointers(L))
    m.set_knobs((0, 0, 2))
    m.run()
    ref = _outs(m)
    m.ctx.set_option(M.MT_OPT_STAGE_SPLIT, 1)
    try:
        for o in m.outputs:
            o.zero_()
        total, stages = m.run()
        for a, b in zip(_outs(m), ref):
            assert torch.equal(a, b)
        assert len(stages) == 4 and all(s > 0 for s in stages)
    finally:
        m.ctx.set_option(M.MT_OPT_STAGE_SPLIT, 0)
    for _ in range(20):
        m.ctx.run_async(m.in_ptrs, m.out_ptrs)
    for a, b in zip(_outs(m), ref):
        assert torch.equal(a, b)
