// Latency microbenchmarks (one warp, one SM sub-partition): dependent chains of the
// SASS instruction kinds on k_decode's event loop.  Each region between two clock
// reads is one dependent chain; scripts/latency_floor.py reads this binary's SASS
// (cuobjdump) to count the chain's instructions per region and divides the printed
// cycles by them, so what ptxas makes of each chain is measured, not assumed.
// Output: "<name> <cycles per link>" lines (a link = one loop-body repetition).
#include <cstdint>
#include <cstdio>

#define N 2048
#define UNROLL 8

#define CHAIN(idx, body)                                                  \
    {                                                                     \
        uint64_t t0 = clock64();                                          \
        for (int i = 0; i < N; ++i) {                                     \
            _Pragma("unroll") for (int u = 0; u < UNROLL; ++u) { body; }  \
        }                                                                 \
        uint64_t t1 = clock64();                                          \
        out[idx] = t1 - t0;                                               \
    }

// one link of the branch chain: LOP3 -> P, a uniform BRA, then 16 dependent IMADs on
// either side (long enough that ptxas keeps the branch instead of predicating)
#define BPAIR(c) "mad.lo.u32 %0, %0, " c ", %2; mad.lo.u32 %0, %0, " c ", %3; "
#define BSIDE(c) BPAIR(c) BPAIR(c) BPAIR(c) BPAIR(c) BPAIR(c) BPAIR(c) BPAIR(c) BPAIR(c) "\n"
#define BLINK(n) "and.b32 t, %0, 1; setp.ne.u32 p, t, 0; @p bra.uni BT" #n ";\n" \
                 BSIDE("%1") "bra.uni BE" #n ";\nBT" #n ": " BSIDE("%4") "BE" #n ":\n"

__global__ void k(uint32_t seed, const uint32_t *__restrict__ cin, uint64_t *out, uint32_t *sink)
{
    __shared__ uint32_t sm[1024];
    const int lane = threadIdx.x;
    for (int i = lane; i < 1024; i += 32) sm[i] = (i * 7 + 1) & 1023;
    __syncwarp();
    // run-time constants the compiler cannot fold
    const uint32_t c0 = cin[0], c1 = cin[1], c2 = cin[2];
    uint32_t v = seed + lane;
    uint64_t x = ((uint64_t)c2 << 32) | v;
    // 0: IADD3 (ptxas merges two adds per IADD3)
    CHAIN(0, asm volatile("add.u32 %0, %0, %1;" : "+r"(v) : "r"(c0)));
    // 1: IMAD
    CHAIN(1, asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(v) : "r"(c0), "r"(c1)));
    // 2: IMAD.HI (the Lemire reciprocal's high products)
    CHAIN(2, asm volatile("mad.hi.u32 %0, %0, %1, %2;" : "+r"(v) : "r"(c0 | 1u), "r"(c1)));
    // 3: IMAD.WIDE.U32 + 64-bit add (T += k * step)
    CHAIN(3, asm volatile("{.reg .u32 lo; cvt.u32.u64 lo, %0; mad.wide.u32 %0, lo, %1, %0;}"
                          : "+l"(x) : "r"(c0)));
    // 4: 64-bit add (IADD3 + IADD3.X)
    CHAIN(4, asm volatile("add.s64 %0, %0, %1;" : "+l"(x) : "l"((uint64_t)c1 << 20 | c0)));
    // 5: ISETP + SEL
    CHAIN(5, asm volatile("{.reg .pred p; setp.gt.u32 p, %0, %1; selp.u32 %0, %2, %1, p;}"
                          : "+r"(v) : "r"(c0), "r"(c1)));
    // 6: 64-bit compare (ISETP + ISETP.EX) + 2 SEL
    CHAIN(6, asm volatile("{.reg .pred p; setp.gt.s64 p, %0, %1; selp.b64 %0, %2, %1, p;}"
                          : "+l"(x) : "l"((uint64_t)c0), "l"((uint64_t)c1 + 7)));
    // 7: LOP3
    CHAIN(7, asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(v) : "r"(c0), "r"(c2)));
    // 8: VIADDMNMX (min + add)
    CHAIN(8, asm volatile("min.u32 %0, %0, %1; add.u32 %0, %0, %2;" : "+r"(v) : "r"(c0), "r"(c1)));
    // 9: CREDUX.MIN -> IMAD.U32 (uniform to vector) -> IMAD.IADD
    CHAIN(9, v = __reduce_min_sync(0xffffffffu, v) + lane);
    // 10: LOP3 -> P, VOTE.ANY, IMAD.IADD
    CHAIN(10, v = __ballot_sync(0xffffffffu, (v >> (lane & 7)) & 1) + lane);
    // 11: ISETP -> P, VOTE.ANY, POPC
    CHAIN(11, v = __popc(__ballot_sync(0xffffffffu, v > (uint32_t)lane)));
    // 12: IMAD.SHL, LOP3, LDS (pointer chase)
    CHAIN(12, v = sm[v & 1023]);
    // 13: IMAD.SHL, LOP3, LDS.64 (pointer chase through an int64 table)
    CHAIN(13, v = (uint32_t)reinterpret_cast<const uint64_t *>(sm)[v & 511] & 1023);
    // 14: uniform data-dependent branch links (see BLINK)
    {
        uint64_t t0 = clock64();
#pragma unroll 1
        for (int i = 0; i < N; ++i) {
            asm volatile("{.reg .pred p; .reg .u32 t;\n"
                         BLINK(0) BLINK(1) BLINK(2) BLINK(3) BLINK(4) BLINK(5) BLINK(6) BLINK(7)
                         "}" : "+r"(v) : "r"(c0), "r"(c1), "r"(c2), "r"(c0 + 2));
        }
        uint64_t t1 = clock64();
        out[14] = t1 - t0;
    }
    sink[lane] = v + (uint32_t)x;
}

int main()
{
    uint64_t *d;
    uint32_t *s, *c;
    cudaMalloc(&d, 64 * 8);
    cudaMalloc(&s, 128);
    cudaMalloc(&c, 16);
    const uint32_t hc[4] = {3u, 0x9E3779B9u, 12345u, 0};
    cudaMemcpy(c, hc, sizeof hc, cudaMemcpyHostToDevice);
    k<<<1, 32>>>(1, c, d, s);
    cudaDeviceSynchronize();
    k<<<1, 32>>>(1, c, d, s);
    cudaDeviceSynchronize();
    uint64_t h[15];
    cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    const char *names[] = {"iadd3", "imad", "imad_hi", "imad_wide", "add64", "isetp_sel",
                           "isetp64_sel64", "lop3", "viaddmnmx", "redux", "vote", "popc_vote",
                           "lds", "lds64", "ubranch"};
    for (int i = 0; i < 15; ++i) printf("%-14s %.3f\n", names[i], h[i] / double(N * UNROLL));
    return 0;
}
