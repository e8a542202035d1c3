"""IR oracle: the paper's unified scheduling IR written out plainly (TEST INFRASTRUCTURE).

Citations are PAPER.md line numbers (P:n) in the paper's §3.2 "Unified Intermediate
Representation Design" and §3.3 "Automated Scheduling Search".

Conventions (readings R1-R4):
  * a tenant's operator sequence is [0, L_i) (0-based; the paper's [1..a], Eq.1);
  * a slice is a half-open range [begin, end); begin == end is the paper's "None" (Eq.5);
  * pointer p means "barrier after operator p" (1-based) == half-open end p (Eq.3);
  * pointer matrix rho[N][P] has the same P for every row (Alg.1 "rho[N, P]") and
    gives P+1 stages ("three sync pointers for four stages"); rows are non-decreasing,
    equal neighbours being empty slices (Eq.5 needs an empty middle slice);
  * an all-empty stage is infeasible ("infeasible solutions ... filtered out").
"""
from __future__ import annotations

from math import comb

# status / error codes (include/mt.h mt_ir_error)
E_OK, E_SHAPE, E_RANGE, E_NONCONTIG, E_EMPTY_STAGE, E_INCOMPLETE, E_ROW_ORDER, E_ROW_RANGE = range(8)

# op kinds (same numbering as include/mt.h; restated here, not imported)
CONV, BN, RELU, MAXPOOL, AVGPOOL, GAP, FC, ADD = 1, 2, 3, 4, 5, 6, 7, 8


def validate(lengths, ranges):
    """Validate a stage-form schedule tau (Eq.6).

    ranges[k][i] = (begin, end) of tenant i in stage k.  Returns the FIRST violation as
    (code, stage, tenant, op) scanning stages k = 0..S-1 and tenants i = 0..N-1, or
    (E_OK, -1, -1, -1).  Checks: Eq.1 order/completeness (every op exactly once, in order:
    contiguous slices starting at 0 and ending at L_i), and no all-empty stage.
    """
    n = len(lengths)
    if len(ranges) < 1 or any(len(st) != n for st in ranges):
        return (E_SHAPE, -1, -1, -1)
    pos = [0] * n
    for k, st in enumerate(ranges):
        all_empty = True
        for i, (b, e) in enumerate(st):
            if b < 0 or e > lengths[i] or b > e:
                return (E_RANGE, k, i, b)
            if b != pos[i]:
                return (E_NONCONTIG, k, i, pos[i])
            if e > b:
                all_empty = False
            pos[i] = e
        if all_empty:
            return (E_EMPTY_STAGE, k, -1, -1)
    for i in range(n):
        if pos[i] != lengths[i]:
            return (E_INCOMPLETE, len(ranges), i, pos[i])
    return (E_OK, -1, -1, -1)


def T(lengths, rho):
    """Schedule generation tau = T(G, rho) (Eq.8).

    Stage k's slice of tenant i is [rho_i[k-1], rho_i[k]) with rho_i[-1] = 0 and
    rho_i[P] = L_i (Eq.3 example: rho_1 = (3,5,7) on [1..10] -> [1,2,3],[4,5],[6,7],[8,9,10]).
    Returns (status_tuple, ranges); ranges is None unless status is E_OK.
    """
    n = len(lengths)
    if len(rho) != n:
        return (E_SHAPE, -1, -1, -1), None
    P = len(rho[0]) if n else 0
    if any(len(r) != P for r in rho):
        return (E_SHAPE, -1, -1, -1), None
    for i, row in enumerate(rho):
        prev = 0
        for k, p in enumerate(row):
            if p < 0 or p > lengths[i]:
                return (E_ROW_RANGE, k, i, p), None
            if p < prev:
                return (E_ROW_ORDER, k, i, p), None
            prev = p
    ranges = []
    for k in range(P + 1):
        st = []
        for i in range(n):
            b = 0 if k == 0 else rho[i][k - 1]
            e = lengths[i] if k == P else rho[i][k]
            st.append((b, e))
        ranges.append(st)
    status = validate(lengths, ranges)
    if status[0] != E_OK:
        return status, None
    return status, ranges


def to_pointers(lengths, ranges):
    """Inverse of T (the 1:1 mapping of P:385): rho_i[k] = end of tenant i's slice in stage k,
    for k = 0..S-2."""
    return [[ranges[k][i][1] for k in range(len(ranges) - 1)] for i in range(len(lengths))]


def stage_of(lengths, ranges):
    """stage_of[i][j] = stage index in which op j of tenant i runs (Eq.4/5 stages)."""
    out = [[-1] * L for L in lengths]
    for k, st in enumerate(ranges):
        for i, (b, e) in enumerate(st):
            for j in range(b, e):
                out[i][j] = k
    return out


def enumerate_schedules(lengths):
    """Every valid schedule, brute force: choose each stage's per-tenant end (>= current
    position) for every possible stage count S = 1..sum(L); keep those passing validate().
    Order: S ascending, then lexicographic in the per-stage end vectors."""
    n = len(lengths)
    total = sum(lengths)
    out = []

    def rec(S, k, pos, acc):
        if k == S:
            if all(p == L for p, L in zip(pos, lengths)):
                out.append([list(st) for st in acc])
            return
        # all end vectors with pos[i] <= e_i <= L_i
        def ends(i, cur):
            if i == n:
                yield list(cur)
                return
            for e in range(pos[i], lengths[i] + 1):
                cur.append(e)
                yield from ends(i + 1, cur)
                cur.pop()
        for ev in ends(0, []):
            if all(e == p for e, p in zip(ev, pos)):
                continue  # all-empty stage
            acc.append([(p, e) for p, e in zip(pos, ev)])
            rec(S, k + 1, ev, acc)
            acc.pop()

    for S in range(1, total + 1):
        rec(S, 0, [0] * n, [])
    return out


def count_schedules(lengths):
    """Closed-form size of the schedule space: for each stage count S, inclusion-exclusion
    over all-empty stages of the product of weak compositions of L_i into S parts:
        count(L) = sum_{S>=1} sum_{j=0}^{S} (-1)^j C(S,j) prod_i W(L_i, S-j),
    W(L, m) = C(L+m-1, m-1) (weak compositions), W(0, 0) = 1, W(L>0, 0) = 0."""
    def W(L, m):
        if m == 0:
            return 1 if L == 0 else 0
        return comb(L + m - 1, m - 1)
    tot = 0
    for S in range(1, sum(lengths) + 1):
        for j in range(S + 1):
            p = 1
            for L in lengths:
                p *= W(L, S - j)
            tot += (-1) ** j * comb(S, j) * p
    return tot


# ----------------------------------------------------------------------------
# Runtime-aware SM partition (north star).  No closed form in the
# paper: "parity unpinned" beyond the invariants tested in tests/test_oracle_ir.py.
# ----------------------------------------------------------------------------

BW_GBS = 8000          # spec HBM bandwidth, GB/s (north star "8 TB/s")
TC_GFLOPS = 2250000    # spec dense bf16 tensor peak, GFLOP/s (2.25 PFLOP/s)


def _numel(c, h, w, batch):
    return batch * c * h * w


def op_cost(graph_nodes, j, batch, in_chw, elem_bytes):
    """(F, B) of op j: F = 2*MACs of conv/FC (0 otherwise), B = bytes of all inputs, weights,
    residual and output at the storage element size (SURVEY §8(d) d.4 'B_op')."""
    nd = graph_nodes[j]

    def chw(i):
        if i == -1:
            return in_chw
        m = graph_nodes[i]
        return (m["out_c"], m["out_h"], m["out_w"])

    ins = [chw(i) for i in nd["inputs"]]
    cin = sum(c for c, _, _ in ins)
    _, h, w = ins[0]
    out_el = _numel(nd["out_c"], nd["out_h"], nd["out_w"], batch)
    in_el = sum(_numel(c, hh, ww, batch) for c, hh, ww in ins)
    k = nd["kind"]
    F = 0
    wel = 0
    if k == CONV:
        macs = out_el * (cin // nd["groups"]) * nd["kh"] * nd["kw"]
        F = 2 * macs
        wel = nd["out_c"] * (cin // nd["groups"]) * nd["kh"] * nd["kw"]
    elif k == FC:
        kin = cin * h * w
        F = 2 * batch * kin * nd["out_c"]
        wel = kin * nd["out_c"]
    res_el = out_el if nd.get("residual", -1) >= 0 else 0
    B = (in_el + wel + res_el + out_el) * elem_bytes
    return F, B


def _largest_remainder(weights, n_sms):
    act = [t for t, w in enumerate(weights) if w is not None]
    out = [0] * len(weights)
    if not act:
        return out
    R = n_sms - len(act)
    ws = {t: weights[t] for t in act}
    W = sum(ws.values())
    if W == 0:
        ws = {t: 1 for t in act}
        W = len(act)
    base = {t: (R * ws[t]) // W for t in act}
    rem = {t: (R * ws[t]) % W for t in act}
    left = R - sum(base.values())
    order = sorted(act, key=lambda t: (-rem[t], t))
    for t in act:
        out[t] = 1 + base[t]
    for t in order[:left]:
        out[t] += 1
    return out


def sm_partition(weights, n_sms, caps=None):
    """Split n_sms CTAs over tenants for one stage, n_t proportional to weights w_t
    (w_t = sum over the tenant's slice of max(F*BW, B*TC), i.e. the slice's roofline time
    scaled by BW*TC), by largest remainder:
        active A = {t : w_t is not None}; R = n_sms - |A|;
        n_t = 1 + floor(R*w_t/W) + [t among the (R - sum floor) largest remainders R*w_t mod W,
              ties to the lower tenant index];   inactive tenants get 0.
    If W == 0 every active tenant weighs 1.
    SURVEY §8(a) a3 tile cap ("n_t <= the max tile count over the slice's ops; any excess is
    redistributed"), caps[t] = that tile count: split over the free tenants U (initially A);
    every tenant of U whose share exceeds its cap is fixed at the cap and leaves U; split the
    SMs left over the new U; repeat.  When every tenant of U exceeds its cap the split over U
    stands (the caps cannot absorb the GPU; reading R16)."""
    out = _largest_remainder(weights, n_sms)
    if caps is None:
        return out
    free = [w is not None for w in weights]
    budget = n_sms
    while True:
        part = _largest_remainder([w if f else None for w, f in zip(weights, free)], budget)
        U = [t for t in range(len(weights)) if free[t]]
        if not U:
            break
        over = [t for t in U if part[t] > caps[t]]
        if not over or len(over) == len(U):
            for t in U:
                out[t] = part[t]
            break
        for t in over:
            out[t] = caps[t]
            budget -= caps[t]
            free[t] = False
    return out


def sm_partition_balanced(items, n_sms, mode=1, hop_ns=2000):
    """Latency-balanced SM partition (reading R16b; not in the paper -- the north
    star's runtime-aware partition with a latency rather than a roofline weight).
    items[t] = None (empty slice) or the list of (tiles, ns) work items of tenant t's slice.
    With n CTAs tenant t needs E_t(n) = sum over its items of ceil(tiles / n) * ns.
    Start: every active tenant 1 CTA.  Then, one CTA at a time, give it to the active tenant
    with the largest E_t among those with n_t < cap_t (cap_t = largest item tile count), ties
    to the lower index; when every active tenant is capped, to the largest E_t regardless.
    Inactive tenants get 0.
    mode 2 (work/span, Brent's bound) instead uses E_t(n) = ceil(W_t / n) + S_t with
    W_t = sum tiles*ns and S_t = sum (ns + hop_ns) over the items."""
    N = len(items)
    out = [0] * N
    act = [t for t in range(N) if items[t] is not None]
    if not act:
        return out

    def E(t, n):
        if mode == 2:
            W = sum(k * ns for k, ns in items[t])
            return -(-W // n) + sum(ns + hop_ns for _, ns in items[t])
        return sum(-(-k // n) * ns for k, ns in items[t])

    cap = {t: max([k for k, _ in items[t]] or [0]) for t in act}
    for t in act:
        out[t] = 1
    for _ in range(n_sms - len(act)):
        cand = [t for t in act if out[t] < cap[t]] or act
        best = max(cand, key=lambda t: (E(t, out[t]), -t))
        out[best] += 1
    return out


def stage_weights(graphs, ranges, elem_bytes_of):
    """Per-stage per-tenant weights for sm_partition (None for an empty slice)."""
    res = []
    for st in ranges:
        row = []
        for t, (b, e) in enumerate(st):
            if b == e:
                row.append(None)
                continue
            g = graphs[t]
            w = 0
            for j in range(b, e):
                F, B = op_cost(g.nodes, j, g.batch, (g.in_c, g.in_h, g.in_w), elem_bytes_of(g))
                w += max(F * BW_GBS, B * TC_GFLOPS)
            row.append(w)
        res.append(row)
    return res
