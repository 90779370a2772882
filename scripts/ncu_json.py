"""profiles/ncu_summary.json from ncu --set full captures: per-launch DRAM
bytes of each hot pass (bench.py's roofline "traffic").
Usage: ncu_json.py TAG  (reads gpurun_out/full_TAG_{HcgA,HcgB,norm_fused}.ncu-rep)"""
import csv
import io
import json
import subprocess
import sys

tag = sys.argv[1]
names = {"HcgA": "hcg_a", "HcgB": "hcg_b", "norm_fused": "norm_b"}
out = {}
for k, key in names.items():
    rep = f"gpurun_out/full_{tag}_{k}.ncu-rep"
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    if len(rows) < 3:
        continue
    h, u, v = rows[0], rows[1], rows[2]
    unit = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1}
    val = lambda m: float(v[h.index(m)].replace(",", "")) * unit.get(u[h.index(m)], 1)  # noqa: E731
    rd, wr = val("dram__bytes_read.sum"), val("dram__bytes_write.sum")
    t = float(v[h.index("gpu__time_duration.sum")].replace(",", ""))
    t_us = t * {"ns": 1e-3, "us": 1.0, "ms": 1e3}.get(u[h.index("gpu__time_duration.sum")], 1.0)
    out[key] = {"kernel": v[h.index("Kernel Name")], "dram_bytes_per_launch": int(rd + wr), "dram_read": int(rd),
                "dram_write": int(wr), "time_us_cold": t_us,
                "dram_pct_peak": float(v[h.index("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed")]),
                "issue_active_pct": float(v[h.index("smsp__issue_active.avg.pct_of_peak_sustained_active")]),
                "capture": f"{rep} (ncu --set full --clock-control none, cd3d 512^3 bf16)"}
json.dump(out, open("profiles/ncu_summary.json", "w"), indent=1)
print(json.dumps({k: (v["dram_bytes_per_launch"], v["time_us_cold"]) for k, v in out.items()}))
