"""Host logic of f4 heterogeneous co-residency (MT_OPT_CTAS_PER_SM = 2), CPU only: option
validation, the plans of the 2-CTA configuration, and the (slot, SM) home pairing rule."""
import numpy as np
import pytest

from workloads import configs

mt = pytest.importorskip("paper_2111_14255_b200.mt")


def _ctx(config, cps):
    g = configs.tenants(config)
    c = mt.Context(-1)
    if cps != 1:
        c.set_option(mt.MT_OPT_CTAS_PER_SM, cps)
    c.load_graphs(g, [[(0x1000, 0x2000, 0x3000) if x.params[j] else None for j in range(x.n_ops)] for x in g])
    return c, g


def test_option_validation():
    c = mt.Context(-1)
    for bad in (0, 3, -1):
        with pytest.raises(mt.MTError):
            c.set_option(mt.MT_OPT_CTAS_PER_SM, bad)
    c.set_option(mt.MT_OPT_CTAS_PER_SM, 2)
    with pytest.raises(mt.MTError) as e:   # fp32 tenants: the SIMT conv tile needs 256 threads
        c.load_graphs(configs.tenants("c1"), [[None] * x.n_ops for x in configs.tenants("c1")])
    assert e.value.status == 3
    c2, _ = _ctx("c2", 2)
    with pytest.raises(mt.MTError) as e:   # plans depend on it: only before loading
        c2.set_option(mt.MT_OPT_CTAS_PER_SM, 1)
    assert e.value.status == 6


def test_two_cta_plans_more_workers_smaller_tiles():
    """the conv cost model sizes tiles for 2 x the CTAs (at least as many tiles per op), the
    CUDA-core tiles shrink with the 128-thread CTA (FC: 4 rows per tile instead of 8)"""
    c1, g = _ctx("c4", 1)
    c2, _ = _ctx("c4", 2)
    n_fc = 0
    for t, gr in enumerate(g):
        for j in range(gr.n_ops):
            p1, p2 = c1.op_plan(t, j), c2.op_plan(t, j)
            assert p1["kind"] == p2["kind"]
            if p1["kind"] == "conv_tc":
                for k in ("path", "tiles_m"):
                    assert p1[k] == p2[k], (gr.name, j, k)
                assert p2["tiles_n"] * p2["splits"] >= p1["tiles_n"] * p1["splits"], (gr.name, j)
            if p1["kind"] == "fc":
                assert p2["tiles"] == 2 * p1["tiles"] or p1["tiles"] % 2, (gr.name, j)
                n_fc += 1
    assert n_fc >= 4


@pytest.mark.parametrize("config", ["c3", "c4"])
def test_home_pairing_rule(config):
    """grid = 2 x #SMs; per stage every tenant owns 2 x its SM share; slot 0 of SM i lists the
    partition from the most to the least compute-intense tenant (FLOP per byte of its slice, from
    mt_op_cost), slot 1 the same list reversed"""
    c, g = _ctx(config, 2)
    L = [x.n_ops for x in g]
    for rho in (configs.all_concurrent_pointers(L), configs.uniform_pointers(L)):
        c.set_schedule_pointers(rho)
        homes, sms = c.stage_homes(), c.sm_partition()
        assert homes.shape[1] == 2 * 148
        ranges = c.get_schedule()
        for k in range(homes.shape[0]):
            h0, h1 = homes[k, :148], homes[k, 148:]
            assert (h1 == h0[::-1]).all()
            for t in range(len(g)):
                assert (homes[k] == t).sum() == 2 * sms[k, t]
            inten = {}
            for t in range(len(g)):
                b, e = ranges[k][t]
                F = B = 0
                for j in range(b, e):
                    f, by = c.op_cost(t, j)
                    F += f
                    B += by
                inten[t] = F / max(B, 1)
            seq = [inten[t] for t in h0]
            assert all(seq[i] >= seq[i + 1] for i in range(len(seq) - 1)), k


def test_one_cta_homes_unchanged():
    c, g = _ctx("c3", 1)
    L = [x.n_ops for x in g]
    c.set_schedule_pointers(configs.all_concurrent_pointers(L))
    homes, sms = c.stage_homes(), c.sm_partition()
    assert homes.shape[1] == 148
    exp = np.concatenate([np.full(sms[0, t], t) for t in range(len(g))])
    assert (homes[0] == exp).all()
