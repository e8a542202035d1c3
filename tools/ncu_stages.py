"""Per-stage ncu counters (SURVEY d.5): summarise a `--set full` capture of a stage-split run
(MT_OPT_STAGE_SPLIT: one executor launch per stage) into profiles/<round>_stage_ncu.json.

  ncu --set full --clock-control none -k regex:executor -s <S*warm> -c <S> -o x python tools/prof_exec.py \\
      --config c3 --schedule uniform4 --stage-split --runs 3
  python tools/ncu_stages.py r01 c3_uniform4=x.ncu-rep
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
WANT = {
    "gpu__time_duration.sum": "duration_us",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed": "tensor_pipe_pct_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct",
}
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "usecond": 1, "us": 1, "msecond": 1e3, "ms": 1e3, "nsecond": 1e-3, "ns": 1e-3}
rnd = sys.argv[1]
out = {}
for arg in sys.argv[2:]:
    key, path = arg.split("=", 1)
    if path.endswith(".csv"):   # an `ncu -i X --page raw --csv` export (made on the GPU box)
        raw = open(path).read()
    else:
        raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    stages = []
    for r in rows[2:]:
        if "executor" not in r[hdr.index("Kernel Name")]:
            continue
        m = {}
        for k, name in WANT.items():
            if k in hdr:
                i = hdr.index(k)
                try:
                    v = float(r[i].replace(",", ""))
                except ValueError:
                    continue
                m[name] = v * UNIT.get(units[i], 1) if name in ("dram_read", "dram_write", "duration_us") else v
        if "dram_read" in m:
            m["dram_bytes"] = int(m.pop("dram_read") + m.pop("dram_write", 0))
        if "duration_us" in m and "dram_bytes" in m:
            m["dram_gbs"] = round(m["dram_bytes"] / (m["duration_us"] * 1e3), 1)
        stages.append(m)
    out[key] = {"source": os.path.basename(path), "stages": stages}
jp = os.path.join(ROOT, "profiles", f"{rnd}_stage_ncu.json")
prev = json.load(open(jp)) if os.path.exists(jp) else {}
prev.update(out)
json.dump(prev, open(jp, "w"), indent=1)
print(json.dumps(out, indent=1))
