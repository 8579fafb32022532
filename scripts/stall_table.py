"""Per-instruction stall samples of the hottest loop in an ncu source-page CSV
(ncu -i X.ncu-rep --page source --csv --print-source sass)."""
import csv
import sys
rows = list(csv.reader(open(sys.argv[1])))
thr = int(sys.argv[2]) if len(sys.argv) > 2 else 50000
hdr = rows[1]
data = rows[2:]
i_s = hdr.index("Warp Stall Sampling (All Samples)")
i_e = hdr.index("Instructions Executed")
stall_cols = [j for j, h in enumerate(hdr) if h.startswith("stall_") or "Stall" in h and "(" not in h]
tot = sum(int(r[i_s]) for r in data)
print("total samples", tot)
hot = 0
for r in data:
    ex = int(r[i_e]) if r[i_e].isdigit() else 0
    if ex > thr:
        hot += int(r[i_s])
        print(r[0][-5:], f"{int(r[i_s]):6d} {ex:8d}", r[1][:72])
print("samples in rows executed >", thr, ":", hot)
