"""Attribute ncu per-SASS warp-stall samples to CUDA source lines.

  python tools/ncu_lines.py gpurun_out/x.ncu-rep [kernel-mangled-name] [--top 40]

Maps SASS offsets to source lines with `nvdisasm -g` on the cubin inside libmt.so (the .so must
be the build that was profiled).
"""
import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
rep = sys.argv[1]
kernel = sys.argv[2] if len(sys.argv) > 2 and not sys.argv[2].startswith("--") else "_ZN3mtk15executor_kernelILb0EEEv7RunArgs"
top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 40
src_csv = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src_csv)))
hdr = rows[1]
ia, isamp = hdr.index("Address"), hdr.index("Warp Stall Sampling (All Samples)")
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
ridx = [hdr.index(h) for h in reasons]
ins = [(int(r[ia], 16), int(r[isamp] or 0), [int(r[k] or 0) for k in ridx]) for r in rows[2:]
       if len(r) > isamp and r[ia].startswith("0x")]
base = ins[0][0]
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.join(ROOT, "paper_2111_14255_b200", "libmt.so")], cwd=tmp,
               capture_output=True)
cubin = [f for f in os.listdir(tmp) if f.startswith("kernels.") and f.endswith(".cubin")][0]
dis = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(tmp, cubin)], capture_output=True, text=True).stdout
line_of = {}
cur = None
infun = False
for ln in dis.splitlines():
    if ln.startswith(".text.") and ln.rstrip().endswith(":"):
        infun = ln.strip()[len(".text."):-1] == kernel
        cur = None
        continue
    if not infun:
        continue
    m = re.search(r'//## File ".*?", line (\d+)', ln)
    if m:
        cur = int(m.group(1))
        continue
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/", ln)
    if m and cur is not None:
        line_of[int(m.group(1), 16)] = cur
src = open(os.path.join(ROOT, "paper_2111_14255_b200", "csrc", "kernels.cu")).read().splitlines()
agg = collections.Counter()
why = collections.defaultdict(lambda: [0] * len(reasons))
tot = 0
for addr, smp, rs in ins:
    off = addr - base
    ln = line_of.get(off, -1)
    agg[ln] += smp
    for k, v in enumerate(rs):
        why[ln][k] += v
    tot += smp
print(f"{rep}: {tot} samples, {len(ins)} SASS instructions")
for line, smp in agg.most_common(top):
    txt = src[line - 1].strip()[:90] if 0 < line <= len(src) else "?"
    w = why[line]
    tw = sum(w) or 1
    top3 = sorted(range(len(w)), key=lambda k: -w[k])[:2]
    rs = " ".join(f"{reasons[k][6:]}:{100 * w[k] // tw}%" for k in top3)
    print(f"{smp:7d} {100.0 * smp / max(tot, 1):5.1f}%  L{line:<5d} {txt[:70]:70s} [{rs}]")
