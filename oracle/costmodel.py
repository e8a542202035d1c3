"""Analytic schedule-cost pre-filter, written out plainly (TEST INFRASTRUCTURE ONLY; only tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline / reference legs may import it).

SURVEY §8(f) f3.  The paper measures the cost of a schedule by profiling and rejects analytic
("modeling-based") costs as inaccurate; this estimate only ranks candidates before
they are profiled.  Form: SPEC.md cost_model's contention model (compute-/memory-time
with linear contention, the longest per-stream chain, a flat per-stage barrier) plus a fixed
latency per dependent operator hop -- DESIGN.md reading R19 (SPEC's examples are inconsistent
with its own normative formula; the normative formula is followed).

estimate(costs, ranges, prm):
    costs[i][j] = (F, B) algorithmic FLOPs / bytes of tenant i's op j (oracle.ir.op_cost);
    ranges[k][i] = (begin, end) of tenant i's slice in stage k (oracle.ir.T);
    prm: dict peak_flops, mem_bw, op_latency_us, sync_us, c_compute, c_memory, max_concurrency.
  roof_j = max(F/peak_flops, B/mem_bw) (us); compute-bound iff F/peak_flops >= B/mem_bw;
  per stage: chain_i = sum_j (roof_j + op_latency_us) over tenant i's slice;
             compute = sum F(compute-bound) / peak * (1 + c_compute * max(0, n_c-1) / max_conc);
             memory  = sum B(memory-bound) / bw   * (1 + c_memory  * max(0, n_m-1) / max_conc);
             stage   = max(compute, memory, max_i chain_i) + sync_us;
  estimate = sum over stages (us).
"""
from __future__ import annotations

US = 1e6


def estimate(costs, ranges, prm):
    peak, bw = prm["peak_flops"], prm["mem_bw"]
    h, sync = prm["op_latency_us"], prm["sync_us"]
    cc, cm = prm.get("c_compute", 0.0), prm.get("c_memory", 0.0)
    mc = max(1, prm.get("max_concurrency", 1))
    total = 0.0
    for stage in ranges:
        C = M = 0.0
        n_c = n_m = 0
        chains = [0.0]
        for i, (b, e) in enumerate(stage):
            chain = 0.0
            has_c = has_m = False
            for j in range(b, e):
                F, B = costs[i][j]
                tc, tm = F / peak * US, B / bw * US
                chain += max(tc, tm) + h
                if tc >= tm:
                    C += F
                    has_c = True
                else:
                    M += B
                    has_m = True
            n_c += has_c
            n_m += has_m
            chains.append(chain)
        compute = C / peak * US * (1.0 + cc * max(0, n_c - 1) / mc)
        memory = M / bw * US * (1.0 + cm * max(0, n_m - 1) / mc)
        total += max(compute, memory, max(chains)) + sync
    return total


def spearman(x, y):
    """Spearman rank correlation (average ranks for ties) -- plain definition"""
    def ranks(v):
        order = sorted(range(len(v)), key=lambda k: v[k])
        r = [0.0] * len(v)
        i = 0
        while i < len(order):
            j = i
            while j + 1 < len(order) and v[order[j + 1]] == v[order[i]]:
                j += 1
            for k in range(i, j + 1):
                r[order[k]] = (i + j) / 2.0 + 1.0
            i = j + 1
        return r
    rx, ry = ranks(list(x)), ranks(list(y))
    n = len(rx)
    mx, my = sum(rx) / n, sum(ry) / n
    cov = sum((a - mx) * (b - my) for a, b in zip(rx, ry))
    vx = sum((a - mx) ** 2 for a in rx) ** 0.5
    vy = sum((b - my) ** 2 for b in ry) ** 0.5
    return cov / (vx * vy) if vx > 0 and vy > 0 else 0.0
