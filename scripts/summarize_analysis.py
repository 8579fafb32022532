"""Summarise the NEXT-row kernels' ncu captures (scripts/prof_analysis.py) into
profiles/<tag>_analysis_ncu.md: launch list shares and one full capture per kernel.

usage: python scripts/summarize_analysis.py <tag> <launches.csv> <full.ncu-rep>
"""
import csv
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag, launches, rep = sys.argv[1:4]
rows = list(csv.reader(open(launches)))
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
d = defaultdict(list)
for r in rows[hdr + 1:]:
    if len(r) > vi and "gl::" in r[ki]:
        d[r[ki].split("(")[0].replace("void ", "")].append(float(r[vi].replace(",", "")))
out = [f"# {tag}: NEXT-row entry points under ncu (`python scripts/prof_analysis.py`: "
       "gl_link_demand on config 4, gl_savings_surface on config 6, gl_complete_matrices on "
       "config 4's Alg. 1 matrices), two calls each", "",
       "## launch list (`--metrics gpu__time_duration.sum --clock-control none`)", "",
       "| kernel | launches | mean us |", "|---|---|---|"]
for k, v in sorted(d.items(), key=lambda kv: -sum(kv[1])):
    out.append(f"| `{k}` | {len(v)} | {sum(v) / len(v) / 1e3:.1f} |")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rr = list(csv.reader(raw.splitlines()))
names, units = rr[0], rr[1]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__t_bytes.sum", "smsp__inst_executed.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size"]
out += ["", "## full captures (`--set full --clock-control none`)", ""]
seen = set()
for vals in rr[2:]:
    kname = vals[names.index("Kernel Name")].split("(")[0]
    if kname in seen:
        continue
    seen.add(kname)
    out.append(f"### `{kname}`")
    for n in want:
        if n in names:
            i = names.index(n)
            out.append(f"- {n}: {vals[i]} {units[i]}")
    st = {n: float(vals[i].replace(",", "") or 0) for i, n in enumerate(names)
          if n.startswith("smsp__pcsamp_warps_issue_stalled_") and not n.endswith("not_issued")}
    tot = sum(st.values()) or 1
    top = sorted(st.items(), key=lambda kv: -kv[1])[:4]
    out.append("- top stalls: " + ", ".join(
        f"{n.replace('smsp__pcsamp_warps_issue_stalled_', '')} {100 * v / tot:.0f}%" for n, v in top))
    out.append("")
open(os.path.join(ROOT, "profiles", f"{tag}_analysis_ncu.md"), "w").write("\n".join(out) + "\n")
print("\n".join(out))
