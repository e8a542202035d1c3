"""Same-box A/B timing of alternative builds of libmt.so (box-to-box variance is ~5%, larger than
most single changes).  Variants are prebuilt .so files; runs alternate variants per config.

  python tools/ab.py --libs ab/A.so,ab/B.so,ab/B.so@2 --configs c2,c3 --rounds 3 --runs 20   (@2: 2 CTAs/SM)
"""
import argparse
import os
import re
import statistics
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ap = argparse.ArgumentParser()
ap.add_argument("--libs", required=True)
ap.add_argument("--configs", default="c2")
ap.add_argument("--rounds", type=int, default=3)
ap.add_argument("--runs", type=int, default=20)
ap.add_argument("--knobs", default="0,0", help="config=rule,depth;... or one rule,depth for all")
a = ap.parse_args()
libs = a.libs.split(",")
res = {}
for r in range(a.rounds):
    for cfg in a.configs.split(","):
        for lib in (libs if r % 2 == 0 else libs[::-1]):
            path, _, cps = lib.partition("@")   # "lib.so@2": run with 2 executor CTAs per SM
            env = dict(os.environ, MT_LIB_PATH=os.path.abspath(path))
            kn = dict(x.split("=") for x in a.knobs.split(";")) if "=" in a.knobs else {}
            out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "prof_exec.py"), "--config", cfg,
                                  "--runs", str(a.runs), "--knobs", kn.get(cfg, a.knobs if not kn else "0,0"),
                                  "--cps", cps or "1"],
                                 capture_output=True, text=True, env=env, timeout=300).stdout
            us = [float(m) for m in re.findall(r"run \d+: ([0-9.]+) us", out)][3:]
            res.setdefault((cfg, lib), []).extend(us)
for cfg in a.configs.split(","):
    row = [f"{cfg:12s}"]
    for lib in libs:
        v = res.get((cfg, lib), [])
        row.append(f"{os.path.basename(lib)}: {statistics.median(v):8.1f} us" if v else f"{lib}: -")
    print("  ".join(row), flush=True)
