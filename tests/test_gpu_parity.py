"""CUDA path (through the C ABI) vs the CPU oracle on a B200.  Run: pytest -m gpu.

Tolerances (north star): fp32 path 1e-4 and bf16 tensor-core path 1e-2 of the output scale
(max |gpu - oracle| / max |oracle|); schedule validity / stage assignment bit-exact (tested on
CPU in test_abi_host.py); outputs bit-identical across every schedule and baseline (P:241-242,
P:314: a schedule changes when operators run, never what they compute)."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import forward as fw  # noqa: E402
from oracle import ir  # noqa: E402
from workloads import configs, zoo  # noqa: E402

from .gpu_helpers import rel_err, teacher_forced_errors  # noqa: E402

_MIXES = {}


def mix_for(config, **kw):
    key = (config, tuple(sorted(kw.items())))
    if key not in _MIXES:
        from paper_2111_14255_b200.session import TenantMix
        graphs = configs.tenants(config, **kw)
        m = TenantMix(graphs)
        x = zoo.make_input(graphs[0])
        m.set_input(x)
        m.x_np = x
        _MIXES[key] = m
    return _MIXES[key]


def _outs(m):
    torch.cuda.synchronize()
    return [o.clone() for o in m.outputs]


# ---------------------------------------------------------------- config 1 (fp32 path, 1e-4)
def test_c1_fp32_hand_schedule_vs_oracle():
    m = mix_for("c1")
    m.ctx.set_schedule_pointers(configs.c1_schedule_pointers())
    total, stages = m.run()
    assert len(stages) == 3 and total > 0 and sum(stages) <= total * 1.0001
    for g, o in zip(m.graphs, m.outputs_numpy()):
        ref = fw.forward(g, m.x_np, "fp32")
        assert rel_err(o, ref) <= 1e-4, g.name
        assert rel_err(o, fw.forward(g, m.x_np, "exact")) <= 1e-4


def test_c1_schedule_invariance_all_287648():
    """EVERY valid schedule of config 1 (the whole 287,648-schedule space of L = (6, 6)) yields
    bit-identical outputs.  Each run writes its own output slot; one
    comparison per chunk of 4096 runs."""
    m = mix_for("c1")
    L = [g.n_ops for g in m.graphs]
    m.ctx.set_schedule_pointers(configs.sequential_pointers(L))
    m.run()
    ref = _outs(m)
    allsch = ir.enumerate_schedules(tuple(L))
    assert len(allsch) == 287648
    CH = 4096
    slots = [torch.empty((CH,) + tuple(o.shape), dtype=o.dtype, device=o.device) for o in m.outputs]
    done = 0
    for c0 in range(0, len(allsch), CH):
        chunk = allsch[c0:c0 + CH]
        for k, s in enumerate(chunk):
            m.ctx.set_schedule(s)
            m.ctx.run_async(m.in_ptrs, [sl[k].data_ptr() for sl in slots])
        torch.cuda.synchronize()
        for sl, r in zip(slots, ref):
            same = (sl[:len(chunk)] == r.unsqueeze(0)).flatten(1).all(dim=1)
            bad = (~same).nonzero().flatten().tolist()
            assert not bad, chunk[bad[0]]
        done += len(chunk)
    assert done == 287648


# ---------------------------------------------------------------- bf16 tensor-core configs
@pytest.mark.parametrize("config", ["c2", "c3", "c4", "c4b8", "f2_models"])
def test_end_to_end_vs_oracle(config):
    m = mix_for(config)
    L = [g.n_ops for g in m.graphs]
    m.ctx.set_schedule_pointers(configs.uniform_pointers(L))
    m.run()
    for g, o in zip(m.graphs, m.outputs_numpy()):
        assert np.isfinite(o).all()
        e_bf = rel_err(o, fw.forward(g, m.x_np, "bf16"))
        assert e_bf <= 1e-2, (g.name, e_bf)


@pytest.mark.parametrize("config", ["c2", "c3", "c4", "c4b8", "f2_models"])
def test_teacher_forced_every_op(config):
    """every op (all 134 conv shapes, dw, pools, FC at b=1 and b=8, concat, residual) recomputed by
    the oracle from the GPU's own bf16 inputs, within 1e-2 of the op's output scale"""
    m = mix_for(config)
    L = [g.n_ops for g in m.graphs]
    m.ctx.set_schedule_pointers(configs.all_concurrent_pointers(L))
    m.run()
    for t, g in enumerate(m.graphs):
        errs = teacher_forced_errors(m, m.x_np, t)
        worst = int(np.argmax(errs))
        assert max(errs) <= 1e-2, (g.name, worst, g.nodes[worst]["kind"], errs[worst])


def test_schedule_and_baseline_invariance_c2():
    m = mix_for("c2")
    L = [g.n_ops for g in m.graphs]
    m.ctx.set_schedule_pointers(configs.all_concurrent_pointers(L))
    m.run()
    ref = _outs(m)
    cands = [configs.sequential_pointers(L), configs.uniform_pointers(L)] + \
        configs.sample_candidates(L, 40, seed=5)[2:]
    n_ok = 0
    for rho in cands:
        try:
            m.ctx.set_schedule_pointers(rho)
        except Exception:
            continue
        n_ok += 1
        m.run()
        for a, b in zip(_outs(m), ref):
            assert torch.equal(a, b), rho
        for mode in ("seq", "ms_dfs", "ms_bfs", "seq_graph", "ms_graph", "stage_events"):
            for o in m.outputs:
                o.zero_()
            m.ctx.run_baseline(mode, m.in_ptrs, m.out_ptrs)
            for a, b in zip(_outs(m), ref):
                assert torch.equal(a, b), (mode, rho)
    assert n_ok >= 30


@pytest.mark.parametrize("config", ["c3", "c4", "c4b8"])
def test_schedule_and_baseline_invariance_large_mixes(config):
    """c3 / c4 / c4b8: both extremes, the uniform split, 256 random candidates (the c5 sampler)
    and all six per-op-launch baselines produce bit-identical outputs (memcmp on the device)."""
    m = mix_for(config)
    L = [g.n_ops for g in m.graphs]
    m.ctx.set_schedule_pointers(configs.all_concurrent_pointers(L))
    m.run()
    ref = _outs(m)
    cands = [configs.sequential_pointers(L), configs.uniform_pointers(L)] + \
        configs.sample_candidates(L, 258, seed=7)[2:]
    n_ok = 0
    for rho in cands:
        try:
            m.ctx.set_schedule_pointers(rho)
        except Exception:
            continue
        n_ok += 1
        for o in m.outputs:
            o.fill_(float("nan"))
        m.ctx.run_async(m.in_ptrs, m.out_ptrs)
        for a, b in zip(_outs(m), ref):
            assert torch.equal(a, b), rho
    assert n_ok >= 250
    m.ctx.set_schedule_pointers(configs.uniform_pointers(L))   # STAGE_EVENTS follows the schedule
    for mode in ("seq", "ms_dfs", "ms_bfs", "seq_graph", "ms_graph", "stage_events"):
        for o in m.outputs:
            o.fill_(float("nan"))
        m.ctx.run_baseline(mode, m.in_ptrs, m.out_ptrs)
        for a, b in zip(_outs(m), ref):
            assert torch.equal(a, b), mode


def test_steal_off_same_outputs():
    from paper_2111_14255_b200.session import TenantMix
    graphs = configs.tenants("c2")
    m1 = mix_for("c2")
    m2 = TenantMix(graphs, steal=False)
    m2.set_input(m1.x_np)
    L = [g.n_ops for g in graphs]
    for mm in (m1, m2):
        mm.ctx.set_schedule_pointers(configs.uniform_pointers(L))
        mm.run()
    for a, b in zip(_outs(m1), _outs(m2)):
        assert torch.equal(a, b)


def test_partition_rules_and_claim_depth_same_outputs():
    """Partition rules (R16/R16b) and bounded claim-ahead change only which CTA runs a tile and
    when: outputs stay bit-identical (c3: three tenants, split-K convs, tensor-core FC)."""
    from paper_2111_14255_b200 import mt as M
    m = mix_for("c3")
    L = [g.n_ops for g in m.graphs]
    for rho in (configs.all_concurrent_pointers(L), configs.uniform_pointers(L)):
        m.ctx.set_schedule_pointers(rho)
        m.ctx.set_option(M.MT_OPT_PARTITION, 0)
        m.ctx.set_option(M.MT_OPT_CLAIM_DEPTH, 0)
        m.run()
        ref = _outs(m)
        for part, steal, depth in ((1, 2, 0), (2, 2, 0), (0, 2, 2), (1, 2, 3), (0, 0, 2), (1, 1, 1)):
            m.ctx.set_option(M.MT_OPT_PARTITION, part)
            m.ctx.set_option(M.MT_OPT_STEAL, steal)
            m.ctx.set_option(M.MT_OPT_CLAIM_DEPTH, depth)
            for o in m.outputs:
                o.zero_()
            m.run()
            for a, b in zip(_outs(m), ref):
                assert torch.equal(a, b), (rho, part, steal, depth)
    m.ctx.set_option(M.MT_OPT_PARTITION, 0)
    m.ctx.set_option(M.MT_OPT_STEAL, 2)
    m.ctx.set_option(M.MT_OPT_CLAIM_DEPTH, 0)
    # Inception's branches: DAG-distance gates (several gate ops per concat consumer)
    m = mix_for("c4")
    L = [g.n_ops for g in m.graphs]
    m.ctx.set_schedule_pointers(configs.all_concurrent_pointers(L))
    m.run()
    ref = _outs(m)
    for depth in (2, 3, 1):
        m.ctx.set_option(M.MT_OPT_CLAIM_DEPTH, depth)
        for o in m.outputs:
            o.zero_()
        m.run()
        for a, b in zip(_outs(m), ref):
            assert torch.equal(a, b), depth
    m.ctx.set_option(M.MT_OPT_CLAIM_DEPTH, 0)


def test_profile_batch_statuses_and_latencies():
    m = mix_for("c2")
    L = [g.n_ops for g in m.graphs]
    cands = configs.sample_candidates(L, 24, seed=9)
    cands.append([[0, 0], [0, 0]])          # all-empty stages -> infeasible
    cands.append([[3, 1], [1, 2]])          # decreasing row -> infeasible
    lat, st = m.ctx.profile_batch_pointers(cands, m.in_ptrs, m.out_ptrs, warmup=1, iters=3)
    for k, rho in enumerate(cands):
        exp_ok = ir.T(L, rho)[0][0] == ir.E_OK
        assert (st[k] == 0) == exp_ok
        if exp_ok:
            assert 1.0 < lat[k] < 1e5
        else:
            assert np.isnan(lat[k])


def test_run_host_matches_device():
    m = mix_for("c2")
    L = [g.n_ops for g in m.graphs]
    m.ctx.set_schedule_pointers(configs.uniform_pointers(L))
    m.run()
    ref = [o.cpu().numpy() for o in _outs(m)]
    xh = torch.from_numpy(m.x_np).pin_memory()
    outs = [torch.empty(o.shape, dtype=torch.float32).pin_memory() for o in m.outputs]
    us = m.ctx.run_host([xh.data_ptr()] * len(L), [o.data_ptr() for o in outs])
    assert us > 0
    for a, b in zip(outs, ref):
        np.testing.assert_array_equal(a.numpy(), b)


def test_unfused_ops_and_pool_variants():
    """standalone BN / RELU / ADD nodes, avg-pool without count_include_pad + ceil_mode, maxpool
    with padding, GAP -> FC, in bf16 and fp32"""
    from paper_2111_14255_b200.session import TenantMix
    for prec, tol in ((zoo.PREC_BF16, 1e-2), (zoo.PREC_FP32, 1e-4)):
        b = zoo.GraphBuilder("tinyA", 2, 3, 19, 17, prec, seed=3)
        x0 = b.conv(-1, 16, 3, 1, 1, act=zoo.ACT_NONE)
        x1 = b.bn(x0)
        x2 = b.relu(x1, act=zoo.ACT_RELU6)
        x3 = b.conv(x2, 16, 1, 1, 0, act=zoo.ACT_RELU)
        x4 = b.add([x2, x3, x1], act=zoo.ACT_RELU)
        x5 = b.avgpool(x4, 3, 2, 1, count_include_pad=False, ceil_mode=True)
        x6 = b.maxpool(x5, 3, 2, 1)
        x7 = b.conv(x6, 24, (1, 3), 1, (0, 1))
        x8 = b.gap(x7)
        b.fc(x8, 10)
        g = b.build()
        m = TenantMix([g])
        x = zoo.make_input(g, seed=4)
        m.set_input(x)
        m.ctx.set_schedule_pointers([[3, 5]])
        m.run()
        mode = "bf16" if prec == zoo.PREC_BF16 else "fp32"
        errs = teacher_forced_errors(m, x, 0)
        assert max(errs) <= tol, errs
        assert rel_err(m.outputs_numpy()[0], fw.forward(g, x, mode)) <= tol


def test_search_drivers_on_gpu_profiler():
    """f1: coordinate descent (Alg.1) and random search through mt_profile_batch; the returned best
    is the best record, and it is never worse than the search's own starting point"""
    from paper_2111_14255_b200 import search
    m = mix_for("c2")
    L = [g.n_ops for g in m.graphs]
    pf = lambda cs: m.ctx.profile_batch_pointers(cs, m.in_ptrs, m.out_ptrs, warmup=1, iters=3)
    cd = search.coordinate_descent(pf, L, P=2, rounds=1, m=4, seed=0)
    assert cd.evaluations == 1 + 1 * 2 * 4
    assert cd.best_lat <= cd.records[0][1] and cd.best_lat == cd.sorted_records()[0][1]
    rs = search.random_search(pf, L, 12, p_max=3, seed=0)
    assert rs.best_rho is not None and np.isfinite(rs.best_lat)
    m.ctx.set_schedule_pointers(cd.best_rho)
    m.run()


def test_operand_path_edge_cases():
    """ragged tensor-core paths: 147-wide rows (column segments 74 + 73) on the 8-channel stem and
    the 64-channel TMA path, strided segments, a tensor-core FC at batch 3 with K % 64 != 0,
    Co % 128 != 0 and a flattened 3x3 spatial input, and the CUDA-core FC after it"""
    from paper_2111_14255_b200.session import TenantMix
    b = zoo.GraphBuilder("tinyA", 3, 3, 147, 147, zoo.PREC_BF16, seed=5)
    x0 = b.conv(-1, 64, 3, 1, 1)                  # stem, 147 wide -> 2 segments
    x1 = b.conv(x0, 64, 3, 1, 1)                  # TMA mode 1, 2 segments, ragged last
    x2 = b.conv(x1, 104, 3, 2, 1)                 # 74 wide, stride 2
    x3 = b.maxpool(x2, 3, 2, 0)                   # 36
    x4 = b.maxpool(x3, 5, 5, 0)                   # 7 x 7 x 104 -> K = 5096 (79.6 k-blocks)
    x5 = b.fc(x4, 200, act=zoo.ACT_RELU)          # b=3 -> tensor-core FC, Co = 200, split-K
    b.fc(x5, 10)
    g = b.build()
    m = TenantMix([g])
    plans = [m.ctx.op_plan(0, j) for j in range(g.n_ops)]
    assert plans[0]["segments"] == 2 and plans[0]["path"] == 2
    assert plans[1]["segments"] == 2 and plans[1]["path"] == 1
    assert plans[5]["path"] == 3 and plans[5]["splits"] > 1     # batch 3: both FCs on tensor cores
    assert plans[6]["path"] == 3
    x = zoo.make_input(g, seed=6)
    m.set_input(x)
    m.ctx.set_schedule_pointers([[2, 5]])
    m.run()
    errs = teacher_forced_errors(m, x, 0)
    assert max(errs) <= 1e-2, errs
    assert rel_err(m.outputs_numpy()[0], fw.forward(g, x, "bf16")) <= 1e-2


def test_wide_n_tiles_bn256():
    """128 x 256 accumulator tiles (TMA path, 256 TMEM columns, 4-stage ring): ragged second N tile
    (Co = 320), fused residual, then a stride-2 conv; per-op teacher-forced vs the oracle at b=8"""
    from paper_2111_14255_b200.session import TenantMix
    b = zoo.GraphBuilder("tinyA", 8, 64, 28, 28, zoo.PREC_BF16, seed=7)
    x0 = b.relu(-1)
    x1 = b.conv(x0, 320, 3, 1, 1)
    x2 = b.conv(x1, 320, 1, 1, 0, residual=x1)
    x3 = b.conv(x2, 512, 3, 2, 1)
    b.fc(b.gap(x3), 10)
    g = b.build()
    m = TenantMix([g])
    plans = [m.ctx.op_plan(0, j) for j in range(g.n_ops)]
    assert plans[1]["bn"] == 256 and plans[2]["bn"] == 256 and plans[1]["tiles_n"] == 2
    x = zoo.make_input(g, seed=8)
    m.set_input(x)
    m.ctx.set_schedule_pointers([[]])
    m.run()
    errs = teacher_forced_errors(m, x, 0)
    assert max(errs) <= 1e-2, errs
    assert rel_err(m.outputs_numpy()[0], fw.forward(g, x, "bf16")) <= 1e-2


def test_stage_split_launches_same_outputs():
    """MT_OPT_STAGE_SPLIT (one launch per stage, SURVEY d.5 profiling mode): identical outputs to
    the single cooperative launch, one stage time per stage, and the counters of the earlier
    launches survive into the later ones (a later stage's ops depend on them)"""
    from paper_2111_14255_b200 import mt as M
    m = mix_for("c3")
    L = [g.n_ops for g in m.graphs]
    m.ctx.set_schedule_pointers(configs.uniform_pointers(L))
    m.run()
    ref = _outs(m)
    m.ctx.set_option(M.MT_OPT_STAGE_SPLIT, 1)
    try:
        for _ in range(2):
            for o in m.outputs:
                o.zero_()
            total, stages = m.run()
            for a, b in zip(_outs(m), ref):
                assert torch.equal(a, b)
            assert len(stages) == 4 and all(s > 0 for s in stages) and total >= sum(stages)
    finally:
        m.ctx.set_option(M.MT_OPT_STAGE_SPLIT, 0)
    m.run()
    for a, b in zip(_outs(m), ref):
        assert torch.equal(a, b)
