"""1-microsecond tick brute-force simulator (an independent formulation).

Pins the oracle (SURVEY.md §8(c.4) "Brute force"): instead of the oracle's
request-ordered recursions and iteration loop, this advances a clock one
microsecond at a time and moves requests between three servers (prefill FCFS
on the new GPU, the stage-2 FIFO, the continuous-batching decode server) under
the written rules R6-R23.  It shares no code with the oracle;
DSD draws use the input module's numpy Philox (a third implementation).
Only for traces whose total time is a few thousand microseconds.
"""
from __future__ import annotations

import math

from paper_2412_20322_b200.inputs.philox import key_from_seed, philox4x32_10

ACCEPT_STREAM = 0x41434350


def _thresholds(alpha, gamma):
    out, x = [], 1.0
    for _ in range(gamma):
        x = x * alpha
        out.append(math.floor(x * 4294967296.0))
    return out


def _draw(seed, j, s):
    k0, k1 = key_from_seed(seed)
    w = philox4x32_10(s // 4, j, ACCEPT_STREAM, 0, k0, k1)
    return int(w[s % 4])


M64 = (1 << 64) - 1


def mix64(j, ttft, finish):
    """SplitMix64 finaliser of j ^ rotl(ttft, 21) ^ rotl(finish, 42)."""
    def rotl(x, k):
        x &= M64
        return ((x << k) | (x >> (64 - k))) & M64
    z = (j ^ rotl(ttft, 21) ^ rotl(finish, 42)) & M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def tick_simulate(trace, ch, t_max=10**6, link=None):
    """``link`` = (bytes_per_token, bytes_per_member_step) records the link
    impulses (R45-R47) as (time, bytes) pairs under "impulses"."""
    if ch.mode >= 2:
        return tick_simulate_colo(trace, ch, t_max)
    bpt, pm = link if link is not None else (0, 0)
    impulses = []
    a = [int(x) for x in trace.arrival_us]
    p = [int(x) for x in trace.prompt_len]
    o = [int(x) for x in trace.output_len]
    n = len(a)
    tb = ch.tables
    thr = _thresholds(ch.alpha, ch.gamma) if ch.mode == 1 else []
    c = [None] * n
    r = [None] * n
    fin = [None] * n
    busy_new = busy_old = e_new = e_old = 0
    arrived = 0
    pf_queue, pf_cur, pf_end = [], None, None
    s2_queue, s2_cur, s2_end = [], None, None
    ready = []               # indices with stage 2 done, in index order
    batch = {}               # j -> [rem, step]
    it_end, it_b = None, 0
    done = 0
    t = 0
    while done < n:
        if t > t_max:
            raise RuntimeError("tick simulation did not terminate")
        changed = True
        while changed:
            changed = False
            while arrived < n and a[arrived] == t:
                pf_queue.append(arrived)
                arrived += 1
                changed = True
            # prefill server
            if pf_cur is not None and pf_end == t:
                j = pf_cur
                c[j] = t
                pf_cur = None
                if o[j] > 1:
                    s2_queue.append(j)
                    if bpt > 0:
                        impulses.append((t, bpt * (p[j] + 1)))
                else:
                    fin[j] = t
                    done += 1
                changed = True
            if pf_cur is None and pf_queue:
                j = pf_queue.pop(0)
                pf_cur, pf_end = j, t + int(tb.t1_us[p[j]])
                busy_new += int(tb.t1_us[p[j]])
                e_new += int(tb.e1_new_uj[p[j]])
                changed = True
            # stage-2 FIFO
            if s2_cur is not None and s2_end == t:
                r[s2_cur] = t
                ready.append(s2_cur)
                s2_cur = None
                changed = True
            if s2_cur is None and s2_queue:
                j = s2_queue.pop(0)
                s2_cur, s2_end = j, t + int(tb.t2_us[p[j]])
                busy_old += int(tb.b2_old_us[p[j]])
                e_old += int(tb.e2_old_uj[p[j]])
                changed = True
        # decode server: iteration boundary at t
        if it_end is not None and it_end == t:
            for j in list(batch):
                if ch.mode == 0:
                    batch[j][0] -= 1
                else:
                    u = _draw(ch.seed, j, batch[j][1])
                    batch[j][0] -= 1 + sum(1 for th in thr if u < th)
                    batch[j][1] += 1
                if batch[j][0] <= 0:
                    fin[j] = t
                    done += 1
                    del batch[j]
            it_end = None
        if it_end is None:
            while ready and len(batch) < ch.cap:
                j = ready.pop(0)
                batch[j] = [o[j] - 1, 0]
            if batch:
                b = len(batch)
                it_end, it_b = t + int(tb.step_us[b]), b
                if pm > 0:
                    impulses.append((t, b * pm))
                busy_new += int(tb.step_busy_new_us[b])
                busy_old += int(tb.step_busy_old_us[b])
                e_new += int(tb.step_e_new_uj[b])
                e_old += int(tb.step_e_old_uj[b])
        t += 1
    ttft = [c[i] - a[i] for i in range(n)]
    ok = 0
    for i in range(n):
        if ttft[i] <= ch.ttft_slo_us and (o[i] == 1 or fin[i] - c[i] <= ch.tpot_slo_us * (o[i] - 1)):
            ok += 1
    return dict(ttft=ttft, finish=fin, ready=r, c=c, slo_ok=ok, busy_new_us=busy_new,
                busy_old_us=busy_old, e_new_uj=e_new, e_old_uj=e_old, tokens=sum(o),
                makespan_us=max(fin), impulses=impulses,
                req_hash=sum(mix64(i, ttft[i], fin[i]) for i in range(n)) & M64)


def window_peak_bruteforce(impulses, window_us):
    """Max over EVERY integer t of the bytes issued in [t, t + window_us), and
    the earliest impulse time whose window attains it (-1 without impulses)."""
    if not impulses:
        return 0, 0, -1
    ts = [t for t, _ in impulses]
    best = 0
    for t0 in range(min(ts) - window_us, max(ts) + 1):
        v = sum(w for t, w in impulses if t0 <= t < t0 + window_us)
        best = max(best, v)
    at = min(t for t in ts if sum(w for u, w in impulses if t <= u < t + window_us) == best)
    return sum(w for _, w in impulses), best, at


def tick_simulate_colo(trace, ch, t_max=10**6):
    """Co-located serving (Standalone, SpecDecode; R41-R44): one GPU that runs
    one job at a time -- a prefill (t1[p]) or one decode iteration at batch b
    (step[b]).  When the GPU frees up at t: finish the job (a prefill's request
    joins the batch, or finishes if o = 1; an iteration's members advance and
    leave), then start the next job: a prefill of the oldest arrived request if
    the batch has room, else an iteration if the batch is non-empty, else idle."""
    a = [int(x) for x in trace.arrival_us]
    p = [int(x) for x in trace.prompt_len]
    o = [int(x) for x in trace.output_len]
    n = len(a)
    tb = ch.tables
    thr = _thresholds(ch.alpha, ch.gamma) if ch.mode == 3 else []
    c = [None] * n
    fin = [None] * n
    busy_new = busy_old = e_new = e_old = 0
    arrived = 0
    queue = []
    batch = {}
    job, job_end = None, None  # ("pf", j) or ("it", b)
    done = 0
    t = 0
    while done < n:
        if t > t_max:
            raise RuntimeError("tick simulation did not terminate")
        while arrived < n and a[arrived] == t:
            queue.append(arrived)
            arrived += 1
        if job is not None and job_end == t:
            if job[0] == "pf":
                j = job[1]
                c[j] = t
                if o[j] > 1:
                    batch[j] = [o[j] - 1, 0]
                else:
                    fin[j] = t
                    done += 1
            else:
                for j in list(batch):
                    if ch.mode == 2:
                        batch[j][0] -= 1
                    else:
                        u = _draw(ch.seed, j, batch[j][1])
                        batch[j][0] -= 1 + sum(1 for th in thr if u < th)
                        batch[j][1] += 1
                    if batch[j][0] <= 0:
                        fin[j] = t
                        done += 1
                        del batch[j]
            job = None
        if job is None:
            if queue and len(batch) < ch.cap:
                j = queue.pop(0)
                job, job_end = ("pf", j), t + int(tb.t1_us[p[j]])
                busy_new += int(tb.t1_us[p[j]])
                e_new += int(tb.e1_new_uj[p[j]])
                if job_end == t:  # zero-length prefill: handle at this tick again
                    continue
            elif batch:
                b = len(batch)
                job, job_end = ("it", b), t + int(tb.step_us[b])
                busy_new += int(tb.step_busy_new_us[b])
                busy_old += int(tb.step_busy_old_us[b])
                e_new += int(tb.step_e_new_uj[b])
                e_old += int(tb.step_e_old_uj[b])
                if job_end == t:
                    continue
        t += 1
    ttft = [c[i] - a[i] for i in range(n)]
    ok = 0
    for i in range(n):
        if ttft[i] <= ch.ttft_slo_us and (o[i] == 1 or fin[i] - c[i] <= ch.tpot_slo_us * (o[i] - 1)):
            ok += 1
    return dict(ttft=ttft, finish=fin, ready=list(a), c=c, slo_ok=ok, busy_new_us=busy_new,
                busy_old_us=busy_old, e_new_uj=e_new, e_old_uj=e_old, tokens=sum(o),
                makespan_us=max(fin),
                req_hash=sum(mix64(i, ttft[i], fin[i]) for i in range(n)) & M64)
