"""Render tools/search_study.py output as profiles/<round>_search.md: the fig:search curves
(best-so-far profiled latency after n evaluations) and the Table III analogue (wall time of the
search at 100 / 300 / 500 / 1000 evaluations).

  python tools/search_report.py gpurun_out/r2j_search.json profiles/r02_search.md
"""
import json
import sys

PAPER = {"alex_vgg_r18": "Alex+VGG+R18", "vgg_r18_r50": "VGG+R18+R50", "r18_r50_r101": "R18+R50+R101"}
MARKS = ("100", "300", "500", "1000")
POINTS = (1, 10, 50, 100, 300, 500, 1000)


def at(curve, n):
    return curve[min(n, len(curve)) - 1] if curve else None


def main(src, dst):
    d = json.load(open(src))
    out = ["# f1 on B200: search curves and search overhead (round 2)", "",
           "`python tools/search_study.py` (one B200): every evaluation is `mt_profile_batch` of one candidate,",
           "W = 2 warm-up + K = 10 timed executor runs, cost = mean device makespan (P:413, P:441).",
           "Knobs (partition rule, claim depth, steal) calibrated per mix first.  Random search = P ~ U{0..8},",
           "rows sorted U{0..L_i} (P:457-461); coordinate descent = Alg.1 with the stage count searched",
           "(P in {0,1,2,3}, M = 8, DESIGN.md R18b); Alg.1 at fixed P = 3 for comparison; naive parallel =",
           "the all-concurrent schedule (one stage, the native scheduler's choice, P:577).", "",
           "## Search overhead (Table III analogue, P:686-709; reading Q11: one round = one evaluation)", "",
           "| mix (paper's name) | method | 100 | 300 | 500 | 1000 evaluations (s) |", "|---|---|---|---|---|---|"]
    for mix, r in d.items():
        for name, key in (("random", "random"), ("coordinate descent over P", "coordinate_descent"),
                          ("Alg.1, P = 3", "coordinate_descent_P3")):
            ts = r[key]["time_s"]
            cells = [f"{ts[m]:.2f}" if ts.get(m) is not None else "-" for m in MARKS]
            out.append(f"| {mix} ({PAPER.get(mix, mix)}) | {name} | " + " | ".join(cells) + " |")
    out += ["", "Paper (Titan V, context only): 9.8 s to 2 min 42 s for 100-1000 rounds (P:702-705).", "",
            "## Best-so-far profiled latency after n evaluations (fig:search analogue, P:663-684), us", "",
            "| mix | naive parallel | sequential | method | " + " | ".join(f"n={p}" for p in POINTS) + " | best |",
            "|---|---|---|---|" + "---|" * len(POINTS) + "---|"]
    for mix, r in d.items():
        fx = r["fixed_us"]
        for name, key in (("random", "random"), ("CD over P", "coordinate_descent"), ("Alg.1 P=3", "coordinate_descent_P3")):
            c = r[key]["curve_us"]
            cells = [f"{at(c, p):.1f}" if at(c, p) is not None and at(c, p) != float("inf") else "-" for p in POINTS]
            best = r[key].get("best_us")
            out.append(f"| {mix} | {fx['naive_parallel']:.1f} | {fx['sequential']:.1f} | {name} | " + " | ".join(cells)
                       + f" | {best:.1f} |")
    out += ["", "Reading: on B200 the persistent executor makes the one-stage (all-concurrent) schedule the best or",
            "within noise of the best on these mixes -- random search and Alg.1 over P converge to it (P = 0);",
            "Alg.1 at a fixed P = 3 cannot reach it (every candidate has 4 stages) and stays 2-9 % slower.",
            "The paper's gains from stage barriers come from contention between host-launched kernels",
            "(P:161-170); the executor removes most of it with dedicated SM groups per tenant and",
            "tile-level dataflow, so barriers can only delay (P:314)."]
    open(dst, "w").write("\n".join(out) + "\n")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
