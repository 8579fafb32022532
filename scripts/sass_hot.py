"""Summarise an ncu report's SASS page: per-instruction stall samples in address order."""
import csv, subprocess, sys
rep = sys.argv[1]
thr = float(sys.argv[2]) if len(sys.argv) > 2 else 0.004
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[1]
ia, isrc = h.index('Address'), h.index('Source')
isamp, iex = h.index('Warp Stall Sampling (All Samples)'), h.index('Instructions Executed')
data = [(int(r[isamp] or 0), int(r[iex] or 0), r[ia][-5:], r[isrc].strip()) for r in rows[2:] if len(r) >= len(h)]
tot = sum(d[0] for d in data)
print("samples", tot, "instructions", sum(d[1] for d in data))
for s, e, a, src in data:
    if s > tot * thr or (len(sys.argv) > 3 and e > 0):
        print(f"{a} {s:6d} {100*s/tot:5.1f}% ex={e:9d}  {src}")
