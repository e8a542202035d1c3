"""C-ABI library on the CPU box: loads, exports every declared symbol, and its host-side plan
compiler (a1-a3) agrees bit for bit with the IR oracle (host-only contexts, no CUDA call)."""
import ctypes as C
import itertools
import random

import numpy as np
import pytest

from oracle import ir
from workloads import configs, zoo

mt = pytest.importorskip("paper_2111_14255_b200.mt")

FAKE = (0x1000, 0x2000, 0x3000)   # host-only contexts never dereference parameter pointers


def host_ctx(graphs, n_sms=148):
    c = mt.Context(-1)
    c.set_option(mt.MT_OPT_NUM_SMS, n_sms)
    c.load_graphs(graphs, [[FAKE if g.params[j] else None for j in range(g.n_ops)] for g in graphs])
    return c


def test_exports_every_declared_symbol():
    names = mt.declared_functions()
    assert len(names) >= 20
    for n in names:
        assert hasattr(mt.lib, n), n
    assert b"sm_100a" in mt.mt_version()


def test_elf_contains_sm100a_tcgen05_code():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", mt.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out
    assert "UTCHMMA" in out or "UTCMMA" in out          # tcgen05.mma
    assert "LDTM" in out                                  # tcgen05.ld


def _tiny_graph(L):
    """a chain of L eltwise ops (8 channels) for IR tests at arbitrary lengths"""
    b = zoo.GraphBuilder("tinyA", 1, 8, 4, 4, zoo.PREC_FP32, seed=0)
    x = -1
    for _ in range(L):
        x = b.relu(x)
    return b.build()


@pytest.mark.parametrize("lengths", [(3, 2), (2, 2, 1), (6, 6)])
def test_validation_bit_exact_on_full_enumeration(lengths):
    """every valid schedule of the space (config 1's (6, 6): all 287,648) through the library:
    accepted, same stage count and op -> stage map as the oracle"""
    c = host_ctx([_tiny_graph(L) for L in lengths])
    sch = ir.enumerate_schedules(lengths)
    assert len(sch) == ir.count_schedules(lengths)
    if lengths == (6, 6):
        assert len(sch) == 287648
    for s in sch:
        c.set_schedule(s)
        assert c.num_stages() == len(s)
        so = c.stage_assignment()
        assert so == ir.stage_of(lengths, s)


def _mutations(lengths, rnd, n):
    out = []
    base = ir.enumerate_schedules(lengths)
    for _ in range(n):
        s = [list(map(list, st)) for st in rnd.choice(base)]
        kind = rnd.randrange(7)
        k = rnd.randrange(len(s))
        i = rnd.randrange(len(lengths))
        if kind == 0:
            s[k][i][1] += rnd.choice([-1, 1])           # overlap / gap / range
        elif kind == 1:
            s[k][i][0] += rnd.choice([-1, 1])
        elif kind == 2 and len(s) > 1:
            s[0], s[-1] = s[-1], s[0]                  # reordered stages
        elif kind == 3:
            s.insert(k, [[st[0], st[0]] for st in s[k]])   # all-empty stage
        elif kind == 4:
            s = s[:-1] if len(s) > 1 else s            # missing ops
        elif kind == 5:
            s[k] = s[k][:-1]                           # wrong N
        else:
            s[k][i] = [s[k][i][1], s[k][i][0]]         # begin > end
        out.append(s)
    return out


def test_validation_errors_bit_exact_on_mutated_corpus():
    lengths = (3, 4, 2)
    c = host_ctx([_tiny_graph(L) for L in lengths])
    rnd = random.Random(7)
    n_err = 0
    for s in _mutations(lengths, rnd, 3000):
        if any(len(st) != len(lengths) for st in s):
            exp = (ir.E_SHAPE, -1, -1, -1)
            arr = None
        else:
            exp = ir.validate(lengths, [[tuple(x) for x in st] for st in s])
        ranges = np.array([x for st in s for x in st], dtype=np.int32).reshape(-1)
        S = len(s) if all(len(st) == len(lengths) for st in s) else 0
        if S == 0:
            st = mt.mt_set_schedule(c.h, 0, ranges.ctypes.data_as(mt.I32P))
        else:
            st = mt.mt_set_schedule(c.h, S, ranges.ctypes.data_as(mt.I32P))
        if exp[0] == ir.E_OK:
            assert st == mt.MT_OK
        else:
            n_err += 1
            assert st == mt.MT_ERR_VALIDATION
            e = mt.mt_error_info()
            mt.mt_last_error_info(c.h, C.byref(e))
            assert (e.code, e.stage, e.tenant, e.op) == exp, (s, exp)
    assert n_err > 1000


def test_pointer_form_bit_exact():
    lengths = (3, 2, 2)
    c = host_ctx([_tiny_graph(L) for L in lengths])
    for P in range(0, 4):
        rows = [list(itertools.combinations_with_replacement(range(-1, L + 2), P)) for L in lengths]
        rnd = random.Random(P)
        for _ in range(400):
            rho = [list(rnd.choice(r)) for r in rows]
            rnd.shuffle(rho[0])
            exp, ranges = ir.T(lengths, rho)
            try:
                c.set_schedule_pointers(rho)
                got = (0, -1, -1, -1)
            except mt.MTError as e:
                assert e.status == mt.MT_ERR_VALIDATION
                got = e.info
            assert got == exp, (rho, got, exp)
            if exp[0] == ir.E_OK:
                assert c.get_schedule().tolist() == [[list(x) for x in st] for st in ranges]


def test_paper_examples_through_abi():
    lengths = (10, 4, 6)
    c = host_ctx([_tiny_graph(L) for L in lengths])
    c.set_schedule_pointers([[3, 5, 7], [1, 2, 3], [2, 2, 4]])
    s = c.get_schedule()
    assert s.shape[0] == 4
    assert s[0].tolist() == [[0, 3], [0, 1], [0, 2]]      # Eq.4 stage 1
    assert s[1].tolist() == [[3, 5], [1, 2], [2, 2]]      # Eq.5 stage 2, S3 None


@pytest.mark.parametrize("config", ["c1", "c2", "c3", "c4", "c4b8"])
def test_op_cost_and_sm_partition_match_oracle(config):
    graphs = configs.tenants(config)
    c = host_ctx(graphs)
    for t, g in enumerate(graphs):
        eb = 2 if g.precision == zoo.PREC_BF16 else 4
        for j in range(g.n_ops):
            assert c.op_cost(t, j) == ir.op_cost(g.nodes, j, g.batch, (g.in_c, g.in_h, g.in_w), eb)
    L = [g.n_ops for g in graphs]
    scheds = [configs.all_concurrent_pointers(L), configs.sequential_pointers(L),
              configs.uniform_pointers(L)] + configs.sample_candidates(L, 40)[2:]
    eb_of = lambda g: 2 if g.precision == zoo.PREC_BF16 else 4
    for rho in scheds:
        st, ranges = ir.T(L, rho)
        if st[0] != ir.E_OK:
            continue
        c.set_schedule_pointers(rho)
        c.set_option(mt.MT_OPT_PARTITION, 0)      # roofline-proportional (north star)
        got = c.sm_partition().tolist()
        caps = [[max([c.op_tiles(t, j) for j in range(b, e)] or [0]) for t, (b, e) in enumerate(st)]
                for st in ranges]   # a3 tile cap: most tiles of one op of the slice
        exp = [ir.sm_partition(w, 148, cp) for w, cp in zip(ir.stage_weights(graphs, ranges, eb_of), caps)]
        assert got == exp
        for mode in (1, 2):                        # latency-balanced (R16b)
            c.set_option(mt.MT_OPT_PARTITION, mode)
            got = c.sm_partition().tolist()
            exp = [ir.sm_partition_balanced([None if b == e else
                                             [it for j in range(b, e) for it in c.op_work(t, j)]
                                             for t, (b, e) in enumerate(st)], 148, mode) for st in ranges]
            assert got == exp
    for t, g in enumerate(graphs):
        for j in range(g.n_ops):
            w = c.op_work(t, j)
            assert sum(k for k, _ in w) == c.op_tiles(t, j) and all(ns > 0 for _, ns in w)


def test_zoo_graphs_ingest_and_reject_bad_graphs():
    for name, f in zoo.MODELS.items():
        g = f()
        c = host_ctx([g])
        assert c.workspace_size() > 0
    g = zoo.resnet18()
    g.nodes[3] = dict(g.nodes[3], out_c=g.nodes[3]["out_c"] + 1)
    with pytest.raises(mt.MTError):
        host_ctx([g])
    g = zoo.resnet18()
    g.nodes[2] = dict(g.nodes[2], inputs=[5])          # not topological
    with pytest.raises(mt.MTError):
        host_ctx([g])


def test_host_only_context_refuses_to_run():
    c = host_ctx([zoo.tinyA()])
    c.set_schedule_pointers([[]])
    with pytest.raises(mt.MTError) as e:
        c.run([0], [0])
    assert e.value.status == mt.MT_ERR_STATE


def test_op_plans_follow_the_operand_rules():
    """mt_op_plan: which path each op takes -- shape + mix only, so the same
    graph gets the same plan whatever the schedule; tiles match mt_op_tiles"""
    c = host_ctx(configs.tenants("c3"))
    vgg = configs.tenants("c3")[1]
    plans = [c.op_plan(1, j) for j in range(vgg.n_ops)]
    assert all(p["tiles"] == c.op_tiles(1, j) for j, p in enumerate(plans))
    assert plans[0]["kind"] == "conv_tc" and plans[0]["path"] == 2 and plans[0]["segments"] == 2   # 8-ch stem, 224 wide
    assert plans[1]["path"] == 1 and plans[1]["segments"] == 2                                    # 224-wide conv: 2 x 112
    assert plans[3]["path"] == 1 and plans[3]["segments"] == 1                                    # 112 wide: whole rows
    fc1 = plans[18]                      # 25088 -> 4096 (205 MB of weights): tensor-core FC, split-K
    assert fc1["kind"] == "conv_tc" and fc1["path"] == 3 and fc1["bn"] == 16 and fc1["tiles_m"] == 32
    assert fc1["splits"] > 1 and fc1["tiles_m"] * fc1["splits"] <= 148
    assert plans[20]["kind"] == "fc"     # 4096 -> 1000 (8.2 MB < 8 MiB): CUDA-core GEMV
    mb = configs.tenants("c3")[2]
    kinds = {c.op_plan(2, j)["kind"] for j in range(mb.n_ops)}
    assert kinds == {"conv_tc", "dw", "gap", "fc"}
    # batch 8: every FC on the tensor-core path
    c8 = host_ctx(configs.tenants("c4b8"))
    for t, g in enumerate(configs.tenants("c4b8")):
        for j, nd in enumerate(g.nodes):
            if nd["kind"] == 7:   # FC
                p = c8.op_plan(t, j)
                assert p["kind"] == "conv_tc" and p["path"] == 3, (g.name, j, p)


def test_scheduling_knob_options_validated():
    """MT_OPT_PARTITION in {0,1,2} re-plans the active schedule; MT_OPT_CLAIM_DEPTH >= 0;
    anything else is MT_ERR_ARG and leaves the previous value (R16b, R20)."""
    graphs = configs.tenants("c2")
    c = host_ctx(graphs)
    L = [g.n_ops for g in graphs]
    c.set_schedule_pointers(configs.all_concurrent_pointers(L))
    c.set_option(mt.MT_OPT_PARTITION, 0)
    p0 = c.sm_partition().tolist()
    c.set_option(mt.MT_OPT_PARTITION, 1)
    p1 = c.sm_partition().tolist()
    assert p0 != p1 and sum(p1[0]) == 148
    for opt, bad in ((mt.MT_OPT_PARTITION, 3), (mt.MT_OPT_PARTITION, -1), (mt.MT_OPT_CLAIM_DEPTH, 1 << 21),
                     (mt.MT_OPT_STAGE_SPLIT, 2)):
        with pytest.raises(Exception):
            c.set_option(opt, bad)
    assert c.sm_partition().tolist() == p1
    for d in (0, 1, 3, 100, -3):
        c.set_option(mt.MT_OPT_CLAIM_DEPTH, d)
    c.set_option(mt.MT_OPT_STAGE_SPLIT, 1)
    c.set_option(mt.MT_OPT_STAGE_SPLIT, 0)
