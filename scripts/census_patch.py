# debug census (A/B only): per-path event counts of the leader's SPL = 1 loop
EDITS = [
("greenllm.cu",
"""int32_t gl_version(void) { return GL_VERSION; }""",
"""int32_t gl_version(void) { return GL_VERSION; }
void gl_census_read(unsigned long long *out, int reset)
{
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(out, gl::gl_census, sizeof(unsigned long long) * 32);
    if (reset) {
        unsigned long long z[32] = {0};
        cudaMemcpyToSymbol(gl::gl_census, z, sizeof z);
    }
}"""),
("k_decode.cuh",
'''namespace gl {

constexpr int DEC_WARPS = 1;''',
'''namespace gl {

__device__ unsigned long long gl_census[32];
#define CEN(i) do { if (ROWS && lane == 0) atomicAdd(&gl_census[i], 1ull); } while (0)

constexpr int DEC_WARPS = 1;'''),
("k_decode.cuh",
'''                const unsigned bit = fr & (0u - fr);
                fr ^= bit;
                const uint32_t fnew = I + h_dj.x;
                if (lane_bit == bit) {
                    Fm = fnew;
                    fa = fin_addr(h_dj.y, nxt);
                }
                fmin = min(fmin, fnew);
                ++b;
                log_b();
                shift_up();
                advance();
            }''',
'''                const unsigned bit = fr & (0u - fr);
                fr ^= bit;
                const uint32_t fnew = I + h_dj.x;
                if (lane_bit == bit) {
                    Fm = fnew;
                    fa = fin_addr(h_dj.y, nxt);
                }
                fmin = min(fmin, fnew);
                ++b;
                log_b();
                shift_up();
                advance();
                CEN(0);  // top join
            }
            CEN(1);  // outer loop trips'''),
("k_decode.cuh",
'''                    if (!(one && h_r <= T && I < 0x80000000u && ((nxt + 2) & 127) > 1 &&
                          (!COLO || h_dj.x != 0))) {
                        if (lv) Fm = F_EMPTY;''',
'''                    if (!(one && h_r <= T && I < 0x80000000u && ((nxt + 2) & 127) > 1 &&
                          (!COLO || h_dj.x != 0))) {
                        if (!one) CEN(14);
                        else if (!(h_r <= T)) CEN(15);
                        else if (((nxt + 2) & 127) <= 1) CEN(16);
                        else CEN(17);
                        if (!one && h_r <= T) CEN(18);  // multi-leave with a ready head
                        if (lv) Fm = F_EMPTY;'''),
("k_decode.cuh",
'''                    prefill();  // co-located: the freed slot's newcomer prefills first
                    fmin = __reduce_min_sync(FULL, Fm);
                    advance_fast();
                }''',
'''                    prefill();  // co-located: the freed slot's newcomer prefills first
                    fmin = __reduce_min_sync(FULL, Fm);
                    advance_fast();
                    CEN(2);  // saturated leave+join
                }
                CEN(3);  // saturated exits'''),
("k_decode.cuh",
'''                        shift_up();
                        advance_fast();
                        if (b == cap || h_r <= T) break;
                    } else {  // leave at iteration fmin (R16)''',
'''                        shift_up();
                        advance_fast();
                        CEN(4);  // light join
                        if (b == cap) { CEN(5); break; }
                        if (h_r <= T) { CEN(6); break; }
                    } else {  // leave at iteration fmin (R16)'''),
("k_decode.cuh",
'''                        if (nl != 1) {  // several members left at once: leave the loop
                            load_nbr(b);
                            break;
                        }
                        if (b == 0 || h_r <= T) break;''',
'''                        CEN(7);  // light leave
                        if (nl != 1) {  // several members left at once: leave the loop
                            CEN(8);
                            load_nbr(b);
                            break;
                        }
                        if (b == 0) { CEN(9); break; }
                        if (h_r <= T) { CEN(10); break; }'''),
("k_decode.cuh",
'''                        if (((nxt + 2) & 127) <= 1) break;  // ring refill due: joins at the top''',
'''                        if (((nxt + 2) & 127) <= 1) { CEN(11); break; }  // ring refill due: joins at the top'''),
("k_decode.cuh",
'''                    if (gap >= 0x80000000ll || I >= 0x80000000u) {
                        slow = true;
                        break;
                    }''',
'''                    if (gap >= 0x80000000ll || I >= 0x80000000u) {
                        CEN(12);
                        slow = true;
                        break;
                    }'''),
("k_decode.cuh",
'''            // ---- general event: a join at kJ < kL, else the leave at kL (R16)
            const int64_t st = st_c;''',
'''            // ---- general event: a join at kJ < kL, else the leave at kL (R16)
            CEN(13);
            const int64_t st = st_c;'''),
]
