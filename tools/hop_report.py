"""Per-op chain latency of one tenant run alone (device trace, tools/trace_exec.py --out X.json):
the op-to-op hop (start of op j+1's first tile -> start of op j+2's first tile, i.e. how fast the
wavefront advances) and, per op, the mean tile phases: dependency wait (claim -> producers
complete), mainloop (-> accumulator ready), epilogue + release.

  python tools/hop_report.py gpurun_out/r2o_trace_r50.json [--md out.md]
"""
import json
import sys

import numpy as np


def main(path, md=None):
    d = json.load(open(path))
    rows = sorted(d["rows"], key=lambda r: r["op"])
    starts = np.array([r["start"] for r in rows])
    hops = np.diff(starts)
    lines = [f"# Chain latency of one tenant alone ({path.split('/')[-1]})", "",
             f"makespan {d['total']:.1f} us, {len(rows)} ops: {d['total'] / len(rows):.2f} us per op; "
             f"op-start hop median {np.median(hops):.2f} us (p10 {np.percentile(hops, 10):.2f}, "
             f"p90 {np.percentile(hops, 90):.2f})", "",
             "| op | tiles | start us | hop us | wait us | mainloop us | epilogue + release us |",
             "|---|---|---|---|---|---|---|"]
    for i, r in enumerate(rows):
        hop = f"{hops[i - 1]:.2f}" if i else "-"
        epi = r["work_mean"] - r["mma_mean"] if r["mma_mean"] > 0 else r["work_mean"]
        ml = f"{r['mma_mean']:.2f}" if r["mma_mean"] > 0 else "-"
        lines.append(f"| {r['name'][:44]} | {r['tiles']} | {r['start']:.1f} | {hop} | {r['wait_mean']:.2f} | {ml} | {epi:.2f} |")
    conv = [r for r in rows if r["mma_mean"] > 0]
    lines += ["", f"conv tiles (mean over ops): wait {np.mean([r['wait_mean'] for r in conv]):.2f} us, mainloop "
              f"{np.mean([r['mma_mean'] for r in conv]):.2f} us, epilogue + release "
              f"{np.mean([r['work_mean'] - r['mma_mean'] for r in conv]):.2f} us"]
    text = "\n".join(lines) + "\n"
    if md:
        open(md, "w").write(text)
    print(text)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[sys.argv.index("--md") + 1] if "--md" in sys.argv else None)
