"""Summarise ncu --set full captures of the executor into profiles/<round>_executor_ncu.json/.md.

  python tools/ncu_summary.py r01 c2=gpurun_out/full_c2.ncu-rep c3=... [launches=gpurun_out/launches.csv]
  (a report may also be given as its `--page raw --csv` export, *.raw.csv)
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
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed": "tensor_pipe_pct_elapsed",
    "sm__pipe_tensor_cycles_active.max.pct_of_peak_sustained_elapsed": "tensor_pipe_pct_max_sm",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
    "launch__registers_per_thread": "registers",
    "launch__grid_size": "grid",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
}
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "usecond": 1, "us": 1, "msecond": 1e3, "ms": 1e3,
        "nsecond": 1e-3, "ns": 1e-3}

rnd = sys.argv[1]
out = {}
for arg in sys.argv[2:]:
    k, path = arg.split("=", 1)
    if k == "launches":
        rows = list(csv.reader(open(path)))
        hdr = next(r for r in rows if r and r[0] == "ID")
        ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
        data = [r for r in rows if r and r[0].isdigit()]
        tot = {}
        for r in data:
            v = float(r[vi].replace(",", "")) * UNIT.get(r[ui], 1)
            name = r[ki].split("(")[0]
            tot[name] = tot.get(name, 0.0) + v
        s = sum(tot.values())
        out["launch_list"] = {"file": os.path.basename(path), "kernels": len(data),
                              "time_share": {n: round(v / s, 4) for n, v in sorted(tot.items(), key=lambda x: -x[1])}}
        continue
    if path.endswith(".csv"):   # an `ncu -i X --page raw --csv` export (made on the GPU box)
        raw = open(path).read()
    else:
        raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        kname = r[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
        if "executor" not in kname:
            continue
        m = {}
        for key, name in WANT.items():
            if key in hdr:
                i = hdr.index(key)
                try:
                    v = float(r[i].replace(",", ""))
                except ValueError:
                    continue
                m[name] = v * UNIT.get(units[i], 1) if name in ("dram_read", "dram_write", "duration_us") else v
        if "dram_read" in m:
            m["dram_bytes_per_launch"] = int(m.get("dram_read", 0) + m.get("dram_write", 0))
        m["source"] = os.path.basename(path)
        out[k] = m
        break
os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
jp = os.path.join(ROOT, "profiles", f"{rnd}_executor_ncu.json")
prev = json.load(open(jp)) if os.path.exists(jp) else {}
prev.update(out)
json.dump(prev, open(jp, "w"), indent=1)
print(json.dumps(prev, indent=1))
