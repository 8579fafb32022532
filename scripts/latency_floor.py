"""Latency floor of k_decode's light-load event loop (bench.py
`roofline.latency`).

Inputs (both reproducible from committed sources):
  * measured dependent-chain latencies: the output of scripts/ubench/lat.cu run on a
    B200 (profiles/<tag>_lat.txt) together with the SASS of that binary (cuobjdump,
    compiled here) -- each timed region's chain instructions are counted in the SASS, so
    the per-instruction latencies below are what the hardware did with what ptxas
    emitted;
  * the SASS of k_decode<1, false, false> from the built libgreenllm.so.

The light loop (decode_run's "light-load fast path", k_decode.cuh) of the LEADER warp is
located in the SASS (the first loop head whose block holds the IMAD.HI.U32 of the
reciprocal ceil-division and whose body stores finish times and reduces with CREDUX), and its two event paths are walked through the control flow:
  J  the head joins at T + kJ * step[b]   (decision branch taken)
  L  one member leaves at iteration fmin  (decision branch not taken, one-leave branch taken)
Every other conditional branch on a path takes its common-case direction (no exit, no
ring refill).  Each path is then timed by two models, over a steady-state alternation
of events with register ready times carried across events:
  dep     dataflow only: an instruction starts when its source registers (and, after a
          conditional branch, the branch's resolution) are ready -- with branches taken
          as free, the loop's minimal dependent-instruction time per event, i.e. the
          latency floor of this SASS (`min_cycles_per_event`);
  inorder the same plus single in-order issue (one instruction per cycle per warp, as a
          warp scheduler issues): a prediction of the loop as it runs.
Output: JSON to stdout (committed as profiles/k_decode_latency.json).

usage: python scripts/latency_floor.py <lat.txt> [--so PATH] [--measured-cycles C]
"""
import argparse
import collections
import json
import os
import re
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KDEC = "_ZN2gl8k_decodeILi1ELb0ELb0EEEvPKNS_6DChainEP14gl_chain_statsPlii"


def sass_lines(binary, fun=None):
    cmd = ["cuobjdump", "-sass"] + (["-fun", fun] if fun else []) + [binary]
    out = subprocess.run(cmd, capture_output=True, text=True).stdout
    res = []
    for ln in out.splitlines():
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s*(.*?)\s*;", ln)
        if m:
            res.append((int(m.group(1), 16), re.sub(r"\s+", " ", m.group(2))))
    # cuobjdump prints the function once per ELF in the fat binary; keep the first copy
    seen, first = set(), []
    for a, s in res:
        if a in seen:
            break
        seen.add(a)
        first.append((a, s))
    return first


def control_stalls(binary, fun):
    """{address: the stall count ptxas encoded in the instruction's control bits} (bits
    41-44 of the high 64-bit word: the cycles the scheduler waits before issuing the
    warp's next instruction, the static part of the schedule)."""
    out = subprocess.run(["cuobjdump", "-sass", "-fun", fun, binary], capture_output=True,
                         text=True).stdout.splitlines()
    res = {}
    for i, ln in enumerate(out):
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s*.*?;\s*/\*\s*0x[0-9a-f]+\s*\*/", ln)
        if not m:
            continue
        a = int(m.group(1), 16)
        if a in res:
            break
        m2 = re.match(r"\s*/\*\s*(0x[0-9a-f]+)\s*\*/", out[i + 1]) if i + 1 < len(out) else None
        if m2:
            res[a] = (int(m2.group(1), 16) >> 41) & 0xF
    return res


def opcode(ins):
    t = ins.split()
    return t[1] if t[0].startswith("@") else t[0]


# ---------------------------------------------------------------- latencies from lat.cu
ALU = {"IADD3", "IADD3.X", "IMAD", "IMAD.IADD", "IMAD.MOV", "IMAD.MOV.U32", "IMAD.SHL.U32",
       "IMAD.U32", "IMAD.X", "MOV", "SEL", "LOP3.LUT", "VIADD", "VIMNMX", "VIMNMX.U32",
       "VIADDMNMX", "VIADDMNMX.U32", "SHF.L.U32", "SHF.R.S32.HI", "SHF.R.U32.HI", "LEA",
       "LEA.HI", "HFMA2", "PLOP3.LUT", "UMOV", "UIADD3", "IADD3.X", "IMAD.HI.U32.X"}


def latencies(lat_txt):
    """Per-instruction latencies (cycles) from the ubench output and its SASS."""
    vals = {}
    for ln in open(lat_txt):
        p = ln.split()
        if len(p) == 2:
            vals[p[0]] = float(p[1])
    with tempfile.TemporaryDirectory() as td:
        exe = os.path.join(td, "lat")
        subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-o", exe,
                        os.path.join(ROOT, "scripts", "ubench", "lat.cu")], check=True,
                       capture_output=True)
        ls = [s for _, s in sass_lines(exe)]
    idx = [i for i, s in enumerate(ls) if "SR_CLOCKLO" in s]
    names = ["iadd3", "imad", "imad_hi", "imad_wide", "add64", "isetp_sel", "isetp64_sel64",
             "lop3", "viaddmnmx", "redux", "vote", "popc_vote", "lds", "lds64", "ubranch"]
    reg, per_link = {}, {}
    for n, a, b in zip(names, idx[0::2], idx[1::2]):
        body = ls[a + 1:b]
        reg[n] = collections.Counter(opcode(s) for s in body)
        # the loop trip counter advances by `inc` source iterations of 8 links each
        inc = [int(m.group(1), 16) for s in body
               for m in [re.match(r"UIADD3 UR\d+, UPT, UPT, UR\d+, (0x[0-9a-f]+), URZ", s)] if m]
        links_per_trip = 8 * inc[0]
        per_link[n] = {op: c / links_per_trip for op, c in reg[n].items()}

    def lat1(name, op):  # cycles per chained instruction of a single-opcode chain
        return vals[name] / per_link[name][op]

    L = {}
    L["alu"] = lat1("imad", "IMAD")
    L["iadd3"] = lat1("iadd3", "IADD3")
    L["lop3"] = lat1("lop3", "LOP3.LUT")
    L["imad_hi"] = lat1("imad_hi", "IMAD.HI.U32")
    # per link: IMAD.WIDE -> IADD3 (low word)
    L["imad_wide"] = vals["imad_wide"] - L["iadd3"]
    # per link: ISETP -> SEL
    L["isetp"] = vals["isetp_sel"] - L["alu"]
    # per link: CREDUX.MIN -> IMAD.U32 (uniform -> vector) -> IMAD.IADD
    L["credux"] = vals["redux"] - 2 * L["alu"]
    # per link: LOP3 (-> P) -> VOTE.ANY -> IMAD.IADD
    L["vote"] = vals["vote"] - L["lop3"] - L["alu"]
    # per link: ISETP -> VOTE.ANY -> POPC
    L["popc"] = vals["popc_vote"] - L["isetp"] - L["vote"]
    # per link: IMAD.SHL -> LOP3 -> LDS
    L["lds"] = vals["lds"] - L["alu"] - L["lop3"]
    L["lds64"] = vals["lds64"] - L["alu"] - L["lop3"]
    # per link: LOP3 (-> P) -> BRA -> 16 dependent IMADs (+ an unconditional BRA on one side)
    L["bra"] = vals["ubranch"] - L["lop3"] - 16 * L["alu"]
    raw = {n: {"cycles_per_link": vals.get(n),
               "sass_per_link": {op: round(v, 3) for op, v in per_link[n].items() if v >= 0.4}}
           for n in names}
    return L, raw


def lat_of(op, L):
    if op.startswith("IMAD.HI"):
        return L["imad_hi"]
    if op.startswith("IMAD.WIDE"):
        return L["imad_wide"]
    if op.startswith("ISETP") or op.startswith("UISETP"):
        return L["isetp"]
    if op.startswith("CREDUX") or op.startswith("REDUX"):
        return L["credux"]
    if op.startswith("VOTE"):
        return L["vote"]
    if op.startswith("POPC"):
        return L["popc"]
    if op.startswith("LDS"):
        return L["lds64"] if ".64" in op or ".128" in op else L["lds"]
    if op.startswith("IADD3"):
        return L["iadd3"]
    if op.startswith("LOP3"):
        return L["lop3"]
    return L["alu"]


# ---------------------------------------------------------------- SASS operand parsing
REG = re.compile(r"^[-~!|]*(U?R\d+|U?P\d+|RZ|PT|URZ|UPT)")


def regs_of(tok, width=1):
    m = REG.match(tok.strip())
    if not m:
        return []
    r = m.group(1)
    if r in ("RZ", "PT", "URZ", "UPT"):
        return []
    if width == 2 and re.match(r"^U?R\d+$", r):
        pre = "UR" if r.startswith("UR") else "R"
        n = int(r[len(pre):])
        return [r, f"{pre}{n + 1}"]
    return [r]


def mem_regs(tok):
    out = []
    for inner in re.findall(r"\[([^\]]*)\]", tok):
        for part in re.split(r"[+\s]", inner):
            w = 2 if part.endswith(".64") else 1
            out += regs_of(part.replace(".64", ""), w)
    return out


def parse(ins):
    """(opcode, dests, srcs, guard, branch_target) of one SASS instruction."""
    t = ins.split(" ", 1)
    guard = None
    if t[0].startswith("@"):
        guard = t[0][1:].lstrip("!")
        t = t[1].split(" ", 1)
    op = t[0]
    ops = [o.strip() for o in t[1].split(",")] if len(t) > 1 else []
    dst, src = [], []
    wide = ".64" in op or ".128" in op
    if not ops:  # operand-less (NOP, DEPBAR, ...)
        return op, [], [], guard, None
    if op.startswith("BRA") or op in ("BSSY", "BSYNC", "EXIT", "NOP") or op.startswith("BSSY") \
            or op.startswith("BSYNC") or op.startswith("WARPSYNC") or op.startswith("YIELD"):
        tgt = None
        for o in ops:
            if o.startswith("0x"):
                tgt = int(o, 16)
            else:
                src += regs_of(o)
        return op, [], src, guard, tgt
    if op.startswith("ST"):
        for i, o in enumerate(ops):
            src += mem_regs(o) if "[" in o else regs_of(o, 2 if wide else 1)
        return op, [], src, guard, None
    if op.startswith("LD"):
        dst += regs_of(ops[0], 2 if wide else 1)
        for o in ops[1:]:
            src += mem_regs(o) if "[" in o else regs_of(o)
        return op, dst, src, guard, None
    if op.startswith("ISETP") or op.startswith("PLOP3") or op.startswith("UISETP"):
        dst += regs_of(ops[0]) + regs_of(ops[1])
        for o in ops[2:]:
            src += regs_of(o)
        return op, dst, src, guard, None
    # generic: operand 0 is the destination; predicate operands right after it are
    # further destinations (carry-outs, LOP3's predicate output ...)
    dst += regs_of(ops[0], 2 if op.startswith("IMAD.WIDE") else 1)
    i = 1
    while i < len(ops) and re.match(r"^(U?P\d+|PT|UPT)$", ops[i]):
        dst += regs_of(ops[i])
        i += 1
    rest = ops[i:]
    for k, o in enumerate(rest):
        w = 2 if (op.startswith("IMAD.WIDE") and k == 2) else 1
        src += regs_of(o, w)
    return op, dst, src, guard, None


# ---------------------------------------------------------------- the light loop's paths
def find_loop(sass):
    """The leader's light loop: the first innermost loop (a branch target t with a
    backward branch to it from past the instruction) around an IMAD.HI.U32 that is
    small (< 200 instructions) and holds both paths: the leave's VOTE / POPC / CREDUX
    and the finish-time store to the rows (STG)."""
    back = collections.defaultdict(list)  # target -> addresses branching back to it
    for a, s in sass:
        tgt = parse(s)[4]
        if tgt is not None and tgt <= a:
            back[tgt].append(a)
    for x, s in sass:
        if opcode(s) != "IMAD.HI.U32":
            continue
        # innermost: the smallest span [t, last back branch] holding x (jumps back from
        # the divergence stubs at the end of the function span far more)
        spans = [(max(srcs) - t, t) for t, srcs in back.items() if t <= x < max(srcs)]
        if not spans:
            continue
        head = min(spans)[1]
        hi = max(back[head])
        body = {opcode(s2) for a2, s2 in sass if head <= a2 <= hi}
        n = sum(1 for a2, _ in sass if head <= a2 <= hi)
        if n < 200 and {"STG.E.64", "CREDUX.MIN", "VOTE.ANY", "POPC"} <= body:
            return head, [a2 for a2, _ in sass]
    raise SystemExit("light loop not found")


def walk(sass, head, decisions, addrs=None):
    """Instructions executed from `head` until the path branches back to `head`
    (their addresses appended to `addrs` if given).
    decisions: one 'T'/'N' per conditional branch met (BRA.DIV: never taken)."""
    pos = {a: i for i, (a, _) in enumerate(sass)}
    i, path, d = pos[head], [], list(decisions)
    while True:
        a, s = sass[i]
        op, dst, src, guard, tgt = parse(s)
        path.append(s)
        if addrs is not None:
            addrs.append(a)
        if op.startswith("BRA"):
            if op == "BRA.DIV":
                taken = False
            elif guard is None:
                taken = True
            else:
                if not d:
                    raise SystemExit(f"path ran out of decisions at {a:#x}: {s}")
                taken = d.pop(0) == "T"
            if taken:
                if tgt == head:
                    if d:
                        raise SystemExit("unused decisions")
                    return path
                i = pos[tgt]
                continue
        i += 1


def simulate(paths, seq, L, inorder, reps=60):
    """Cycles per event of a repeated event sequence (steady state)."""
    ready = collections.defaultdict(float)
    t_issue, t_ctrl = 0.0, 0.0
    times = []
    for r in range(reps):
        for ev in seq:
            for ins in paths[ev]:
                op, dst, src, guard, tgt = parse(ins)
                srcs = src + ([guard] if guard else [])
                t = max([ready[x] for x in srcs] + [t_ctrl])
                if inorder:
                    t = max(t, t_issue + 1.0)
                t_issue = t
                if op.startswith("BRA"):
                    if guard is not None and op != "BRA.DIV":
                        t_ctrl = t + L["bra"]  # later instructions wait for the resolution
                    elif op == "BRA":
                        t_ctrl = t + L["bra"] / 2  # unconditional jump: a fetch redirect
                    continue
                for x in dst:
                    ready[x] = t + lat_of(op, L)
            times.append(t_issue)
    n = len(seq)
    half = reps // 2
    return (times[-1] - times[half * n - 1]) / ((reps - half) * n)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("lat")
    ap.add_argument("--so", default=os.path.join(ROOT, "paper_2412_20322_b200", "libgreenllm.so"))
    ap.add_argument("--measured-cycles", type=float, default=None,
                    help="achieved cycles per event of the critical chain (bench)")
    ap.add_argument("--crit", action="append", default=[],
                    help="cfgN:chain:kernel_ms:decode_requests:sm_mhz -- a config's critical chain "
                         "(one launch of that chain alone), reported with its cycles per event")
    ap.add_argument("--loop-measured", action="append", default=[],
                    help="cfgN:cycles -- the light loop's measured cycles per event "
                         "(scripts/loop_stalls.py on an ncu source-level capture)")
    ap.add_argument("--join", default="NTNT", help="branch decisions of the J path")
    ap.add_argument("--leave", default="NNTT", help="branch decisions of the L path")
    a = ap.parse_args()
    L, raw = latencies(a.lat)
    sass = sass_lines(a.so, KDEC)
    head, _ = find_loop(sass)
    addrs = {"J": [], "L": []}
    paths = {"J": walk(sass, head, a.join, addrs["J"]), "L": walk(sass, head, a.leave, addrs["L"])}
    ctl = control_stalls(a.so, KDEC)
    res = {"source": "scripts/latency_floor.py: measured latencies (scripts/ubench/lat.cu on a B200) "
                     "along the SASS of k_decode<1,0,0>'s leader light-load loop",
           "latencies_cycles": {k: round(v, 2) for k, v in L.items()},
           "ubench": raw, "loop_head": hex(head),
           "paths": {k: {"instructions": len(v), "sass": v} for k, v in paths.items()}}
    # branch resolution: the ubench's figure (LOP3 -> P -> BRA -> IMAD, the predicate
    # written just before the branch) is an upper bound -- with it the in-order model
    # overshoots the measured loop -- so the floor takes branches as free and the
    # in-order view is reported both ways
    for label, bra in (("no_branch_cost", 0.0), ("ubench_branch_cost", L["bra"])):
        L2 = dict(L, bra=bra)
        res[label] = {m: {"J_alone": round(simulate(paths, "J", L2, m == "inorder"), 1),
                          "L_alone": round(simulate(paths, "L", L2, m == "inorder"), 1),
                          "JL_alternating": round(simulate(paths, "JL", L2, m == "inorder"), 1)}
                      for m in ("dep", "inorder")}
    # the critical chain alternates join / leave: the floor is the alternating sequence's
    # dataflow time with free branches (the loop's minimal dependent-instruction cycles)
    # the schedule ptxas encoded: control-code stall counts summed along each path (the
    # static part of the issue time; scoreboard waits on LDS / VOTE / REDUX come on top)
    res["scheduled_stalls"] = {k: sum(ctl.get(x, 0) for x in v) for k, v in addrs.items()}
    res["scheduled_stalls"]["JL_mean"] = (res["scheduled_stalls"]["J"] + res["scheduled_stalls"]["L"]) / 2
    res["min_cycles_per_event"] = res["no_branch_cost"]["dep"]["JL_alternating"]
    res["issue_bound_cycles_per_event"] = res["no_branch_cost"]["inorder"]["JL_alternating"]
    if a.measured_cycles:
        res["measured_cycles_per_event"] = a.measured_cycles
        res["frac"] = round(res["min_cycles_per_event"] / a.measured_cycles, 3)
    crit = {}
    for c in a.crit:
        cfg, chain, ms, m, mhz = c.split(":")
        cyc = float(ms) * 1e-3 * float(mhz) * 1e6 / (2 * int(m))
        crit[cfg] = {"chain": int(chain), "kernel_ms_alone": float(ms), "decode_requests": int(m),
                     "sm_mhz": float(mhz), "cycles_per_event": round(cyc, 1),
                     "frac": round(res["min_cycles_per_event"] / cyc, 3)}
    for c in a.loop_measured:
        cfg, cyc = c.split(":")
        crit.setdefault(cfg, {})["light_loop_cycles_per_event"] = float(cyc)
        crit[cfg]["light_loop_frac"] = round(res["min_cycles_per_event"] / float(cyc), 3)
    if crit:
        res["critical_chain"] = crit
    res["command"] = "python scripts/latency_floor.py " + " ".join(sys.argv[1:])
    json.dump(res, sys.stdout, indent=1)
    print()


if __name__ == "__main__":
    main()
