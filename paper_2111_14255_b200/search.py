"""Schedule search drivers on top of mt_profile_batch (§3.3).

The cost of a candidate is its profiled latency -- "profile the latency by multiple runs" (Alg.1 L8,
P:413), "the averaged latency is then used as the cost" -- measured by the library on the GPU
(`profile_fn`, e.g. Context.profile_batch_pointers).  Infeasible candidates come back with a non-zero
status and are "filtered out".  Both searches keep the record dictionary D{schedule: cost}
(Alg.1 L3/L9) and return the globally best record (L14-15).

  random_search       -- "samples scheduling solutions (different pointer matrices) randomly from the
                         search space ... a memory module will record all schedules"
  coordinate_descent  -- Alg.1: rows of rho are coordinates; for each row sample M
                         candidates, profile them, keep the argmin row; R rounds

Readings (R13, R20): a pointer row is a non-decreasing P-vector in [0, L_i]; coordinate
descent starts from the uniform split (the all-concurrent matrix is infeasible for P > 0 because its
later stages would be empty) and evaluates the start point once (the "+1" of SPEC S:331); ties go to
the earlier evaluation.
"""
from __future__ import annotations

import random
from dataclasses import dataclass, field

import numpy as np


@dataclass
class SearchResult:
    best_rho: list
    best_lat: float
    records: list = field(default_factory=list)     # [(rho, lat, status)] in evaluation order
    evaluations: int = 0

    def sorted_records(self):
        """Alg.1 L14: records sorted by profiled latency (feasible only)"""
        ok = [r for r in self.records if r[2] == 0 and np.isfinite(r[1])]
        return sorted(ok, key=lambda r: r[1])


def _sample_row(rng: random.Random, L: int, P: int):
    return sorted(rng.randint(0, L) for _ in range(P))


def _record(res: SearchResult, cands, lat, st):
    for rho, l, s in zip(cands, lat, st):
        res.records.append(([list(r) for r in rho], float(l), int(s)))
        res.evaluations += 1
        if s == 0 and np.isfinite(l) and l < res.best_lat:
            res.best_lat = float(l)
            res.best_rho = [list(r) for r in rho]


def random_search(profile_fn, lengths, n_candidates: int, p_max: int = 8, seed: int = 0,
                  batch: int = 256) -> SearchResult:
    rng = random.Random(seed)
    res = SearchResult(best_rho=None, best_lat=float("inf"))
    todo = []
    for _ in range(n_candidates):
        P = rng.randint(0, p_max)
        todo.append([_sample_row(rng, L, P) for L in lengths])
    for k in range(0, len(todo), batch):
        chunk = todo[k:k + batch]
        lat, st = profile_fn(chunk)
        _record(res, chunk, lat, st)
    return res


def coordinate_descent(profile_fn, lengths, P: int, rounds: int, m: int, seed: int = 0,
                       init=None) -> SearchResult:
    """Alg.1.  Evaluations = 1 + rounds * N * m."""
    rng = random.Random(seed)
    n = len(lengths)
    rho = [list(r) for r in init] if init is not None else \
        [[(2 * k * L + (P + 1)) // (2 * (P + 1)) for k in range(1, P + 1)] for L in lengths]
    res = SearchResult(best_rho=None, best_lat=float("inf"))
    lat, st = profile_fn([rho])
    _record(res, [rho], lat, st)
    for _ in range(rounds):                       # L4
        for i in range(n):                        # L5
            cands = []
            for _ in range(m):                    # L6: M candidate rows for row i
                c = [list(r) for r in rho]
                c[i] = _sample_row(rng, lengths[i], P)
                cands.append(c)
            lat, st = profile_fn(cands)          # L7-L8: profile each
            _record(res, cands, lat, st)          # L9: append to D
            ok = [k for k in range(m) if st[k] == 0 and np.isfinite(lat[k])]
            if ok:                                # L11: keep the row with the lowest latency
                kbest = min(ok, key=lambda k: (lat[k], k))
                rho = cands[kbest]
    return res                                    # L14-15: global best of D


def coordinate_descent_over_p(profile_fn, lengths, p_values, rounds: int, m: int,
                              seed: int = 0) -> SearchResult:
    """Alg.1 with the stage count searched too (R18b): Alg.1 fixes P (rho[N, P]),
    so with a fixed P > 0 it can never return a schedule with fewer stages -- the all-concurrent
    schedule (P = 0) in particular, whose matrix has no pointers at all.  For every P of p_values
    (ascending) run Alg.1 (P = 0 is its single candidate); D collects every evaluation and the
    global best of D is returned (L14-15).  Evaluations = sum over P of (1 + rounds * N * m) for
    P > 0, 1 for P = 0."""
    res = SearchResult(best_rho=None, best_lat=float("inf"))
    for k, P in enumerate(p_values):
        if P == 0:
            rho = [[] for _ in lengths]
            lat, st = profile_fn([rho])
            _record(res, [rho], lat, st)
            continue
        r = coordinate_descent(profile_fn, lengths, P, rounds, m, seed=seed + k)
        for rho, l, s in r.records:
            _record(res, [rho], [l], [s])
    return res


def prefiltered_search(estimate_fn, profile_fn, candidates, keep: int) -> SearchResult:
    """rank `candidates` by the analytic estimate (estimate_fn(cands) -> (est,
    status), e.g. Context.estimate_batch_pointers; microseconds of host time per candidate), then
    profile only the `keep` best-estimated feasible ones -- the cost stays the profiled latency
    (P:441).  Returns the SearchResult of the profiled subset; `records` holds only those."""
    est, est_st = estimate_fn(candidates)
    ok = [k for k in range(len(candidates)) if est_st[k] == 0 and np.isfinite(est[k])]
    ok.sort(key=lambda k: (est[k], k))
    chosen = [candidates[k] for k in ok[:keep]]
    res = SearchResult(best_rho=None, best_lat=float("inf"))
    if chosen:
        lat, st = profile_fn(chosen)
        _record(res, chosen, lat, st)
    return res
