"""Source edits for scripts/ab_build.py: name -> [(file, old, new), ...]."""

LIGHT_HEAD_OLD = '''                    const int64_t gap = h_r - T;
                    const uint32_t kJ = ceil_div_magic((uint32_t)gap, (uint32_t)st, M_c);
                    if (gap >= 0x80000000ll || I >= 0x80000000u) {
                        slow = true;
                        break;
                    }
                    if (kJ < kL) {  // the head joins at T + kJ * step[b]
                        T += (int64_t)kJ * st;'''

VARIANTS = {
    "base": [],
    # the rare far-gap / rebase check only on the join branch (clamped kJ)
    "clamp": [("k_decode.cuh", LIGHT_HEAD_OLD, '''                    const int64_t gap = h_r - T;
                    const uint32_t kJ = ceil_div_magic(
                        (uint32_t)min(gap, (int64_t)0x7FFFFFFF), (uint32_t)st, M_c);
                    if (kJ < kL) {  // the head joins at T + kJ * step[b]
                        if (gap >= 0x80000000ll || I >= 0x80000000u) {
                            slow = true;
                            break;
                        }
                        T += (int64_t)kJ * st;''')],
    # join/leave decided by a warp vote: a uniform predicate needs no reconvergence
    "vote": [("k_decode.cuh", '''                    if (kJ < kL) {  // the head joins at T + kJ * step[b]
                        T += (int64_t)kJ * st;''', '''                    if (__all_sync(FULL, kJ < kL)) {  // the head joins at T + kJ * step[b]
                        T += (int64_t)kJ * st;''')],
    # multi-leave test from the ballot directly (no popc on the branch)
    "lm": [("k_decode.cuh", '''                        const int nl = __popc(lm);
                        b -= nl;
                        log_b();
                        mk = T;
                        fmin = __reduce_min_sync(FULL, Fm);
                        if (nl == 1) shift_down();
                        else load_nbr(b);
                        if (b == 0 || h_r <= T) break;''', '''                        const int nl = __popc(lm);
                        b -= nl;
                        log_b();
                        mk = T;
                        fmin = __reduce_min_sync(FULL, Fm);
                        if ((lm & (lm - 1u)) == 0u) shift_down();
                        else load_nbr(b);
                        if (b == 0 || h_r <= T) break;''')],
}
