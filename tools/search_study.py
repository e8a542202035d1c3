"""SURVEY §8(f) f1 evidence on B200: the search curves of fig:search (§4.4) and the
search-overhead table (Table III) for the paper's three mixes, profiled through
mt_profile_batch (W=2, K=10 per candidate; the cost is the averaged measured latency).

  random search          -- P:457-461 (P ~ U{0..8}, rows sorted U{0..L_i})
  coordinate descent     -- Alg.1, stage count searched too (R18b), M = 8
  naive parallel         -- all-concurrent schedule (one stage): the native scheduler
  sequential             -- one tenant per stage

For each: best-so-far latency after n evaluations and the wall time to reach n = 100 / 300 /
500 / 1000 evaluations (Table III's rounds, reading Q11: one round = one evaluated candidate).

  python tools/search_study.py [--mixes alex_vgg_r18,vgg_r18_r50,r18_r50_r101] [--evals 1000]
      [--out gpurun_out/search_study.json]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2111_14255_b200 import search as S  # noqa: E402
from paper_2111_14255_b200.session import TenantMix  # noqa: E402
from workloads import configs, zoo  # noqa: E402

PAPER_T3 = {   # Table III (Titan V): search time at 100 / 300 / 500 / 1000 rounds -- context only
    "alex_vgg_r18": "Alex+VGG+R18", "vgg_r18_r50": "VGG+R18+R50", "r18_r50_r101": "R18+R50+R101"}
MARKS = (100, 300, 500, 1000)


class Recorder:
    """wraps the profiler: per evaluation (in order) its latency, status and the wall time at
    which its batch returned"""

    def __init__(self, fn):
        self.fn = fn
        self.t0 = time.perf_counter()
        self.lat, self.st, self.t = [], [], []

    def __call__(self, cands):
        lat, st = self.fn(cands)
        now = time.perf_counter() - self.t0
        self.lat += [float(v) for v in lat]
        self.st += [int(v) for v in st]
        self.t += [now] * len(cands)
        return lat, st

    def curve(self, n):
        best, out = float("inf"), []
        for l, s in zip(self.lat[:n], self.st[:n]):
            if s == 0 and np.isfinite(l):
                best = min(best, l)
            out.append(best)
        return out

    def time_at(self, n):
        return self.t[n - 1] if len(self.t) >= n else None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mixes", default="alex_vgg_r18,vgg_r18_r50,r18_r50_r101")
    ap.add_argument("--evals", type=int, default=1000)
    ap.add_argument("--out", default="gpurun_out/search_study.json")
    a = ap.parse_args()
    sp = torch.cuda.current_stream().cuda_stream
    res = {}
    for mix in a.mixes.split(","):
        g = configs.tenants(mix)
        L = [x.n_ops for x in g]
        m = TenantMix(g)
        m.set_input(zoo.make_input(g[0]))
        knobs, _ = m.calibrate()
        prof = lambda cs: m.ctx.profile_batch_pointers(cs, m.in_ptrs, m.out_ptrs, 2, 10, sp)
        prof([configs.all_concurrent_pointers(L)] * 4)   # warm
        r = {"tenants": list(configs.CONFIGS[mix][0]), "ops": L, "knobs": list(knobs)}
        fixed = {}
        for name, rho in (("naive_parallel", configs.all_concurrent_pointers(L)),
                          ("sequential", configs.sequential_pointers(L))):
            lat, st = prof([rho])
            fixed[name] = float(lat[0])
        r["fixed_us"] = fixed
        # random search (batches of 50 so the curve's time stamps are fine-grained)
        rec = Recorder(prof)
        S.random_search(rec, L, a.evals, p_max=8, seed=14255, batch=50)
        r["random"] = {"curve_us": rec.curve(a.evals), "time_s": {n: rec.time_at(n) for n in MARKS},
                       "best_us": min(rec.curve(a.evals))}
        # coordinate descent over P = 0..3 with enough rounds to spend ~a.evals evaluations
        M = 8
        per_round = len(L) * M
        R = max(1, (a.evals - 1) // (3 * per_round))
        rec = Recorder(prof)
        cd = S.coordinate_descent_over_p(rec, L, (0, 1, 2, 3), rounds=R, m=M, seed=14255)
        n = len(rec.lat)
        r["coordinate_descent"] = {"rounds": R, "m": M, "evaluations": n, "curve_us": rec.curve(n),
                                   "time_s": {k: rec.time_at(k) for k in MARKS}, "best_us": cd.best_lat,
                                   "best_P": len(cd.best_rho[0])}
        # fixed-P Alg.1 (P = 3) for reference: cannot reach fewer stages
        rec = Recorder(prof)
        cd3 = S.coordinate_descent(rec, L, P=3, rounds=max(1, (a.evals - 1) // per_round), m=M, seed=14255)
        r["coordinate_descent_P3"] = {"evaluations": len(rec.lat), "curve_us": rec.curve(len(rec.lat)),
                                      "time_s": {k: rec.time_at(k) for k in MARKS}, "best_us": cd3.best_lat}
        res[mix] = r
        print(f"{mix}: naive {fixed['naive_parallel']:.1f} seq {fixed['sequential']:.1f} | random best "
              f"{r['random']['best_us']:.1f} (t@1000 {r['random']['time_s'][1000]}) | CD best {cd.best_lat:.1f} "
              f"P={len(cd.best_rho[0])} ({n} evals) | CD P=3 best {cd3.best_lat:.1f}", flush=True)
        del m
        torch.cuda.empty_cache()
    json.dump(res, open(a.out, "w"))


if __name__ == "__main__":
    main()
