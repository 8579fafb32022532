"""Summarise ncu outputs from gpurun_out/ into profiles/ (committed evidence).

usage: python scripts/summarize_profiles.py <round tag> <launches.csv> <kernel.ncu-rep> [kernel]
"""
import csv
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag, launches, rep = sys.argv[1], sys.argv[2], sys.argv[3]
kern = sys.argv[4] if len(sys.argv) > 4 else "k_decode"
out_dir = os.path.join(ROOT, "profiles")

# ---- launch list: per-kernel count, mean device time, share of the step
rows = list(csv.reader(open(launches)))
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
d = defaultdict(list)
for r in rows[hdr + 1:]:
    if len(r) > vi:
        d[r[ki]].append(float(r[vi].replace(",", "")))
ours = {k: v for k, v in d.items() if "gl::" in k}
tot = sum(sum(v) for v in ours.values())
lines = [f"# {tag}: ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, "
         f"serialised launches) of `python bench.py --steps 3 --warmup 3`", "",
         "| kernel | launches | mean us | share of our kernels' time |", "|---|---|---|---|"]
for k, v in sorted(ours.items(), key=lambda kv: -sum(kv[1])):
    name = k.split("(")[0].replace("void ", "")
    lines.append(f"| `{name}` | {len(v)} | {sum(v) / len(v) / 1e3:.1f} | {sum(v) / tot:.4f} |")
other = {k: v for k, v in d.items() if k not in ours}
if other:
    lines.append("")
    lines.append("Other (PyTorch) launches in the same run: " +
                 ", ".join(f"{k.split('(')[0][:60]} x{len(v)}" for k, v in other.items()))
open(os.path.join(out_dir, f"{tag}_launches.md"), "w").write("\n".join(lines) + "\n")

# ---- full capture of the dominant kernel
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rr = list(csv.reader(raw.splitlines()))
names, units, vals = rr[0], rr[1], rr[2]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__t_bytes.sum", "lts__t_sectors.sum", "lts__t_requests.sum",
        "smsp__inst_executed.sum", "sm__inst_executed.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
        "sm__cycles_elapsed.avg", "smsp__cycles_active.avg"]
m = {}
for i, n in enumerate(names):
    if n in want or n.startswith("smsp__pcsamp_warps_issue_stalled_"):
        m[n] = (vals[i], units[i])
lines = [f"# {tag}: `ncu --set full --clock-control none --import-source on -k regex:{kern}` "
         "on `python bench.py --steps 1 --warmup 3` (config 4, 64 chains x 100k requests)", ""]
for n in want:
    if n in m:
        lines.append(f"- {n}: {m[n][0]} {m[n][1]}")
lines.append("")
lines.append("Warp-stall samples (PC sampling):")
stalls = {n: float(v[0].replace(",", "")) for n, v in m.items()
          if n.startswith("smsp__pcsamp_warps_issue_stalled_") and not n.endswith("not_issued")}
tot_s = sum(stalls.values()) or 1
for n, v in sorted(stalls.items(), key=lambda kv: -kv[1]):
    if v > 0:
        lines.append(f"- {n.replace('smsp__pcsamp_warps_issue_stalled_', '')}: {v:.0f} "
                     f"({100 * v / tot_s:.1f}%)")
open(os.path.join(out_dir, f"{tag}_{kern}_ncu.md"), "w").write("\n".join(lines) + "\n")


def num(n):
    v, u = m[n]
    v = float(v.replace(",", ""))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
    return v * scale


dram = num("dram__bytes_read.sum") + num("dram__bytes_write.sum")
l2 = num("lts__t_sectors.sum") * 32 if "lts__t_sectors.sum" in m else None
json.dump({"round": tag, "kernel": kern, "dram_bytes_per_launch": dram,
           "l2_bytes_per_launch": l2,
           "warp_inst_per_launch": num("smsp__inst_executed.sum"),
           "source": f"profiles/{tag}_{kern}_ncu.md"},
          open(os.path.join(out_dir, f"{kern}_dram_bytes.json"), "w"), indent=1)
print(open(os.path.join(out_dir, f"{tag}_launches.md")).read())
print(open(os.path.join(out_dir, f"{tag}_{kern}_ncu.md")).read())
