"""Pins of the IR oracle (oracle/ir.py) against the paper's worked examples, closed forms,
brute force and invariants -- none of which re-type the oracle's own formulas."""
import itertools
import json
import os

import pytest

from oracle import ir

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_ir_examples.json")))


def _inclusive(b, e):
    """half-open 0-based [b, e) -> the paper's 1-based inclusive [b+1, e] or None"""
    return None if b == e else [b + 1, e]


def test_eq3_pointer_split():
    ex = GOLD["eq3"]
    st, ranges = ir.T([ex["length"]], [ex["pointers"]])
    assert st[0] == ir.E_OK
    assert [_inclusive(*s[0]) for s in ranges] == ex["segments"]


def test_eq4_eq5_stages():
    ex = GOLD["eq4_eq5"]
    st, ranges = ir.T(ex["lengths"], ex["rho"])
    assert st[0] == ir.E_OK
    assert len(ranges) == ex["n_stages"]
    assert [_inclusive(*s) for s in ranges[0]] == ex["stage1"]
    assert [_inclusive(*s) for s in ranges[1]] == ex["stage2"]


def test_round_trip_pointers():
    ex = GOLD["eq4_eq5"]
    _, ranges = ir.T(ex["lengths"], ex["rho"])
    assert ir.to_pointers(ex["lengths"], ranges) == ex["rho"]


@pytest.mark.parametrize("lengths,expected", [
    ((1, 1), 3), ((2, 2), 26), ((2, 3), 76), ((3, 3), 252), ((4, 4), 2568),
    ((3, 3, 3), 64324), ((2, 2, 2, 2), 47834), ((6, 6), 287648), ((1,), 1), ((4,), 8),
])
def test_count_closed_form_values(lengths, expected):
    # (4,) -> 2^3 = 8 compositions of 4; others SURVEY c.4 [DERIVED]
    assert ir.count_schedules(lengths) == expected


@pytest.mark.parametrize("lengths", [(1, 1), (2, 2), (2, 3), (3, 3), (1, 2, 2), (4,), (3, 1, 2)])
def test_enumeration_matches_closed_form_and_is_valid(lengths):
    sch = ir.enumerate_schedules(lengths)
    assert len(sch) == ir.count_schedules(lengths)
    keys = {repr(s) for s in sch}
    assert len(keys) == len(sch)
    for s in sch:
        assert ir.validate(lengths, s)[0] == ir.E_OK


@pytest.mark.parametrize("lengths", [(2, 2), (2, 3), (1, 2, 2)])
def test_T_is_bijection_onto_valid_schedules(lengths):
    """Image of T over ALL fixed-P non-decreasing pointer matrices (P = 0..sum L - 1) equals the
    brute-force enumeration, and T is injective on feasible matrices (the 1:1 map)."""
    target = {repr(s) for s in ir.enumerate_schedules(lengths)}
    image = {}
    for P in range(sum(lengths)):
        rows = [list(itertools.combinations_with_replacement(range(L + 1), P)) for L in lengths]
        for rho in itertools.product(*rows):
            rho = [list(r) for r in rho]
            st, ranges = ir.T(lengths, rho)
            if st[0] != ir.E_OK:
                assert st[0] == ir.E_EMPTY_STAGE
                continue
            key = repr(ranges)
            assert key not in image, "T not injective"
            image[key] = rho
    assert set(image) == target


def test_spec_strict_subspace_count():
    """lengths (3,3), <=1 strictly-increasing pointer per row in 1..L-1 -> 9 matrices,
    all feasible under T once padded to a common P (pad with L_i)."""
    lengths = (3, 3)
    cnt = 0
    for r0 in ([], [1], [2]):
        for r1 in ([], [1], [2]):
            P = max(len(r0), len(r1))
            rho = [r0 + [3] * (P - len(r0)), r1 + [3] * (P - len(r1))]
            st, _ = ir.T(lengths, rho)
            assert st[0] == ir.E_OK
            cnt += 1
    assert cnt == 9


def test_extremes_valid_and_enumerated():
    from workloads import configs
    lengths = (2, 3, 1)
    allc = configs.all_concurrent_pointers(lengths)
    seq = configs.sequential_pointers(lengths)
    st, r_all = ir.T(lengths, allc)
    assert st[0] == ir.E_OK and len(r_all) == 1
    st, r_seq = ir.T(lengths, seq)
    assert st[0] == ir.E_OK and len(r_seq) == len(lengths)
    for k, stage in enumerate(r_seq):  # stage k = tenant k alone
        for i, (b, e) in enumerate(stage):
            assert (b < e) == (i == k)
    enum = {repr(s) for s in ir.enumerate_schedules(lengths)}
    assert repr(r_all) in enum and repr(r_seq) in enum


@pytest.mark.parametrize("ranges,expected", [
    ([], (ir.E_SHAPE, -1, -1, -1)),
    ([[(0, 2)]], (ir.E_SHAPE, -1, -1, -1)),                            # wrong N
    ([[(0, 2), (0, 1)], [(2, 2), (1, 4)]], (ir.E_RANGE, 1, 1, 1)),     # end > L
    ([[(0, 1), (0, 3)], [(2, 3), (3, 3)]], (ir.E_NONCONTIG, 1, 0, 1)),  # gap
    ([[(0, 2), (0, 3)], [(1, 3), (3, 3)]], (ir.E_NONCONTIG, 1, 0, 2)),  # overlap
    ([[(0, 2), (0, 3)], [(2, 2), (3, 3)], [(2, 3), (3, 3)]], (ir.E_EMPTY_STAGE, 1, -1, -1)),
    ([[(0, 2), (0, 2)]], (ir.E_INCOMPLETE, 1, 0, 2)),                  # missing op
    ([[(2, 3), (0, 3)], [(0, 2), (3, 3)]], (ir.E_NONCONTIG, 0, 0, 0)),  # reordered stages
    ([[(1, 0), (0, 3)], [(0, 3), (3, 3)]], (ir.E_RANGE, 0, 0, 1)),      # begin > end
])
def test_validation_mutations(ranges, expected):
    assert ir.validate((3, 3), ranges) == expected


def test_pointer_row_errors():
    assert ir.T((3, 3), [[2, 1], [1, 2]])[0] == (ir.E_ROW_ORDER, 1, 0, 1)
    assert ir.T((3, 3), [[1, 4], [1, 2]])[0] == (ir.E_ROW_RANGE, 1, 0, 4)
    assert ir.T((3, 3), [[1], [1, 2]])[0][0] == ir.E_SHAPE
    assert ir.T((3, 3), [[1, 1], [1, 1]])[0] == (ir.E_EMPTY_STAGE, 1, -1, -1)


def test_stage_of_partition_of_ops():
    lengths = (10, 4, 6)
    _, ranges = ir.T(lengths, GOLD["eq4_eq5"]["rho"])
    so = ir.stage_of(lengths, ranges)
    for i, L in enumerate(lengths):
        assert len(so[i]) == L
        assert so[i] == sorted(so[i])             # dependency order preserved across stages
        assert all(0 <= s < len(ranges) for s in so[i])
    assert so[2][2] == 2 and so[2][1] == 0        # S_3 empty in stage 2 (index 1)


def test_sm_partition_invariants_and_hand_examples():
    assert ir.sm_partition([1, 1], 148) == [74, 74]
    # R = 146: 146*3/4 = 109 r2, 146*1/4 = 36 r2 -> tie -> lower index takes the extra SM
    assert ir.sm_partition([3, 1], 148) == [111, 37]
    assert ir.sm_partition([None, 5, None], 148) == [0, 148, 0]
    assert ir.sm_partition([0, 0], 10) == [5, 5]
    assert ir.sm_partition([10**17, 1], 148) == [147, 1]
    import random
    rnd = random.Random(3)
    for _ in range(500):
        n = rnd.randint(1, 6)
        w = [None if rnd.random() < 0.2 else rnd.randint(0, 10**15) for _ in range(n)]
        out = ir.sm_partition(w, 148)
        act = [t for t in range(n) if w[t] is not None]
        if not act:
            assert out == [0] * n
            continue
        assert sum(out) == 148
        W = sum(w[t] for t in act)
        for t in range(n):
            if w[t] is None:
                assert out[t] == 0
            else:
                assert out[t] >= 1
                if W:
                    ideal = 1 + (148 - len(act)) * w[t] / W
                    assert abs(out[t] - ideal) < 1.0 + 1e-9


def _E(items, t, n, mode, hop=2000):
    if mode == 2:   # Brent: work / n + span
        return -(-sum(k * ns for k, ns in items[t]) // n) + sum(ns + hop for _, ns in items[t])
    return sum(-(-k // n) * ns for k, ns in items[t])


def _minimax_brute(items, n_sms, mode=1):
    """exhaustive optimum of max_t E_t(n_t) over every split of n_sms (each active tenant >= 1)"""
    act = [t for t in range(len(items)) if items[t] is not None]

    def E(t, n):
        return _E(items, t, n, mode)

    best = None

    def rec(i, left, acc):
        nonlocal best
        if i == len(act) - 1:
            v = max(acc + [E(act[i], left)])
            best = v if best is None else min(best, v)
            return
        for n in range(1, left - (len(act) - 1 - i) + 1):
            rec(i + 1, left - n, acc + [E(act[i], n)])

    rec(0, n_sms, [])
    return best


def test_sm_partition_balanced_is_the_minimax_optimum():
    """R16b: greedy 'feed the current maximum' reaches the exact minimum over all splits of
    max_t sum ceil(tiles/n_t)*ns (brute force on small instances), keeps the invariants, and
    reduces to an even split for identical tenants."""
    import random
    rnd = random.Random(11)
    assert ir.sm_partition_balanced([[(100, 10)], [(100, 10)]], 10) == [5, 5]
    # one long chain of 1-tile ops needs 1 CTA; the wide op gets the rest
    assert ir.sm_partition_balanced([[(1, 1000)] * 5, [(64, 100)]], 9) == [1, 8]
    assert ir.sm_partition_balanced([None, [(3, 1)], None], 7) == [0, 7, 0]
    for _ in range(300):
        n = rnd.randint(1, 4)
        items = [None if rnd.random() < 0.2 else
                 [(rnd.randint(1, 40), rnd.randint(1, 5000)) for _ in range(rnd.randint(1, 4))]
                 for _ in range(n)]
        act = [t for t in range(n) if items[t] is not None]
        n_sms = rnd.randint(max(1, len(act)), 14)
        for mode in (1, 2):
            out = ir.sm_partition_balanced(items, n_sms, mode)
            if not act:
                assert out == [0] * n
                continue
            assert sum(out) == n_sms
            assert all((out[t] >= 1) == (items[t] is not None) for t in range(n))
            got = max(_E(items, t, out[t], mode) for t in act)
            assert got == _minimax_brute(items, n_sms, mode)
