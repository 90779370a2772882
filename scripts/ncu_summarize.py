"""Text summary of an ncu --set full report (key metrics, stall reasons, top
stalled SASS lines) for profiles/.  Usage: ncu_summarize.py REPORT [TITLE]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
title = sys.argv[2] if len(sys.argv) > 2 else rep


def run(*a):
    return subprocess.run(["ncu", "-i", rep, *a], capture_output=True, text=True).stdout


rows = list(csv.reader(io.StringIO(run("--page", "raw", "--csv"))))
h, u, v = rows[0], rows[1], rows[2]
want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "lts__t_sector_hit_rate.pct",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "launch__shared_mem_per_block_dynamic", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum"]
print(f"# ncu summary: {title}\n\nsource: `{rep}` (ncu --set full --clock-control none --import-source on)\n")
print("| metric | value | unit |\n|---|---|---|")
for w in want:
    if w in h:
        i = h.index(w)
        print(f"| {w} | {v[i][:100]} | {u[i]} |")
st = [(h[i], float(v[i] or 0)) for i in range(len(h))
      if h[i].startswith("smsp__average_warps_issue_stalled_") and h[i].endswith("_per_issue_active.ratio")]
st.sort(key=lambda x: -x[1])
print("\n## warp stall reasons (warps per issue)\n\n| reason | ratio |\n|---|---|")
for k, val in st[:10]:
    print(f"| {k.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')} | {val:.3f} |")
src = list(csv.reader(io.StringIO(run("--page", "source", "--csv", "--print-source", "sass"))))
if len(src) > 2:
    hh = src[1]
    si, sx = hh.index("Warp Stall Sampling (All Samples)"), hh.index("Source")
    data = [r for r in src[2:] if len(r) > si and r[si].isdigit()]
    tot = sum(int(r[si]) for r in data) or 1
    print(f"\n## top stalled SASS instructions ({tot} samples)\n\n| share | instruction |\n|---|---|")
    for r in sorted(data, key=lambda r: -int(r[si]))[:12]:
        print(f"| {100 * int(r[si]) / tot:.1f}% | `{r[sx].strip()[:90]}` |")
