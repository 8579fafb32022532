"""Measured stall samples along the leader's light-load loop (ncu source page of one
chain's k_decode launch, e.g. `ncu --set full --import-source on ... python
scripts/prof_chains.py 33`) next to scripts/latency_floor.py's in-order model of the
same SASS.  Prints a markdown report: per instruction of the join (J) and leave (L)
paths the executions, the warp-stall samples and their main reasons, and the
light loop's measured cycles per event (its samples' share of the launch x the
launch's cycles / its events) against the model's floor and in-order figures.

usage: python scripts/loop_stalls.py <kernel.ncu-rep> <lat.txt> <kernel_ms> <sm_mhz> [title]
"""
import collections
import csv
import io
import os
import subprocess
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__))))
import latency_floor as lf  # noqa: E402

REASONS = ["stall_wait", "stall_selected", "stall_branch_resolving", "stall_short_sb",
           "stall_dispatch", "stall_no_inst", "stall_not_selected", "stall_mio", "stall_math",
           "stall_long_sb", "stall_lg"]


def main():
    rep, lat, kms, mhz = sys.argv[1], sys.argv[2], float(sys.argv[3]), float(sys.argv[4])
    title = sys.argv[5] if len(sys.argv) > 5 else rep
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[1]
    isrc, isamp, iex = h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), \
        h.index("Instructions Executed")
    irs = {r: h.index(r) for r in REASONS if r in h}
    data = [r for r in rows[2:] if len(r) >= len(h)]
    def norm(s):  # SASS text without branch targets (ncu prints absolute addresses)
        t = " ".join(s.replace(";", "").split())
        return " ".join(w for w in t.split() if not w.startswith("0x7f")) if "BRA" in t else t
    so = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                      "paper_2412_20322_b200", "libgreenllm.so")
    sass = lf.sass_lines(so, lf.KDEC)
    head, _ = lf.find_loop(sass)
    pos = {a: i for i, (a, _) in enumerate(sass)}
    # the CSV lists the function's instructions in address order, as cuobjdump does
    def same(i):  # ncu and cuobjdump print operands slightly differently: opcodes match
        return lf.opcode(norm(data[i][isrc])) == lf.opcode(norm(sass[i][1]))
    assert len(data) == len(sass) and all(same(i) for i in range(len(sass))), \
        "ncu rows do not match the SASS of the built library"
    total = sum(int(r[isamp] or 0) for r in data)
    cyc_per_sample = kms * 1e-3 * mhz * 1e6 / max(total, 1)
    L, _ = lf.latencies(lat)
    paths = {"J": lf.walk(sass, head, "NTNT"), "L": lf.walk(sass, head, "NNTT")}
    # instruction indices on each path, in path order (a path revisits no address)
    idx = {}
    for k in "JL":
        i, lst, d = pos[head], [], list("NTNT" if k == "J" else "NNTT")
        for ins in paths[k]:
            while sass[i][1] != ins:
                i += 1
            lst.append(i)
            op, _, _, guard, tgt = lf.parse(ins)
            if op.startswith("BRA") and op != "BRA.DIV" and (guard is None or d.pop(0) == "T"):
                if tgt == head:
                    break
                i = pos[tgt]
                continue
            i += 1
        idx[k] = lst
    loop_ids = sorted(set(idx["J"]) | set(idx["L"]))
    ev_j = int(data[idx["J"][-1]][iex] or 0)  # J's loop-back branch
    ev_l = int(data[idx["L"][-1]][iex] or 0)  # L's loop-back branch
    s_loop = sum(int(data[i][isamp] or 0) for i in loop_ids)
    reason_tot = collections.Counter()
    for i in loop_ids:
        for r, j in irs.items():
            reason_tot[r] += int(data[i][j] or 0)
    meas = s_loop * cyc_per_sample / max(ev_j + ev_l, 1)
    L0 = dict(L, bra=0.0)
    dep = lf.simulate(paths, "JL", L0, False)
    ino = lf.simulate(paths, "JL", L0, True)
    print(f"# {title}\n")
    print(f"Launch {kms} ms at {mhz:.0f} MHz = {kms * 1e-3 * mhz * 1e6 / 1e6:.1f} M cycles, "
          f"{total} warp-stall samples ({cyc_per_sample:.0f} cycles per sample).  The leader's "
          f"light loop (loop head at SASS offset {hex(head)}): {s_loop} samples "
          f"({100 * s_loop / total:.1f}% of the launch) over {ev_j} join and {ev_l} leave events "
          f"(executions of each path's loop-back branch, ncu).\n")
    print("| light loop | cycles per event |\n|---|---|")
    print(f"| measured (samples x cycles per sample / events) | {meas:.1f} |")
    print(f"| model, in-order issue, branches free | {ino:.1f} |")
    print(f"| model, dataflow floor, branches free (`min_cycles_per_event`) | {dep:.1f} |")
    print(f"| floor / measured | {dep / meas:.3f} |\n")
    print("Stall reasons over the loop's samples: " + ", ".join(
        f"{r[6:]} {100 * v / max(sum(reason_tot.values()), 1):.0f}%"
        for r, v in reason_tot.most_common() if v) + "\n")
    for k in "JL":
        print(f"## {k} path ({len(idx[k])} instructions)\n")
        print("| offset | executions | samples | main stall reasons | SASS |\n|---|---|---|---|---|")
        for i in idx[k]:
            r = data[i]
            rs = sorted(((int(r[j] or 0), n[6:]) for n, j in irs.items()), reverse=True)
            top = ", ".join(f"{n} {v}" for v, n in rs[:2] if v)
            print(f"| {sass[i][0]:#06x} | {int(r[iex] or 0)} | {int(r[isamp] or 0)} | {top} | "
                  f"`{norm(sass[i][1])}` |")
        print()


if __name__ == "__main__":
    main()
