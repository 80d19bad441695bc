// hash_tiled_bs.cu -- WMH_ALGO_TILED for dense rows, bit-sliced tile (default).
//
// Same draws, same result as the other tiles (the draw stream of hash j does
// not depend on x, so one draw serves every row of the tile), but
// the tile is stored as BIT PLANES: for column c and a group of 32 rows, NB
// words whose bit i is bit b of x[row i][c] (NB = bits of the largest bound).
// Alg. 5's test for one draw (c, off) and all 32 rows of a group is then the
// carry out of the bit-serial sum x + L, L = 2^NB - 1 - off:
//
//   green(x)  <=>  x > off  <=>  x + L >= 2^NB
//   carry_{b+1} = MAJ(x_b, L_b, carry_b)     (one LOP3 per bit, 32 rows at once)
//
// with L_b as an all-ones / all-zeros mask (one PRMT sign-replicate of a word
// holding L's bits at byte MSBs).  About 2*NB + 8 instructions test a draw
// against 32 rows -- against ~2 per row for the byte-SWAR tile.
//
// A warp takes one hash for the whole tile (G groups of 32 rows): lane =
// (group, part), each lane draws DPL consecutive t of the group's round, the
// parts of a group combine their green masks with a segmented prefix OR, and
// the first green t of each pending row is recorded (h = t + 1, Alg. 3 / Def.,
// P:166-188).  Rows stay pending until green or the cap (h = cap, reading R9);
// all-zero rows never turn green and get the cap at once (R12).
#include <stdio.h>
#include <stdlib.h>

#include <type_traits>
#include <vector>

#include "common.cuh"

namespace wmh {

constexpr int BS_NT = 512;
constexpr int BS_NW = BS_NT / 32;
constexpr int BS_HB = 8;                 // hashes per claimed block (results flushed 8 per row)
// draws per lane per round by groups per tile (a round of a group = 32 / G
// lanes x DPL draws): longer rounds amortise the per-round scan and test
// setup against draws tested past a group's last first-green.  Measured on
// c5 (G = 2): DPL 2 / 4 / 8 -> 334 / 313 / 329 ms; on c2 (G = 4): 4 beats 8
// (0.75 vs 0.81 ms)
__host__ __device__ constexpr int bs_dpl(int G) { return G == 1 ? 2 : G == 2 ? 4 : G == 4 ? 4 : 8; }

struct BsParams {
    const uint8_t *x;
    int64_t n_rows;
    int D, G;                    // dim, groups of 32 rows per tile
    int n_hchunks, hchunk;
    int64_t n_items;
    uint32_t k, cap, M, uni_m;
    uint64_t S;
    int vec_flush, sigb;
    const uint32_t *table;       // [k][T0] (c * G * NBS) << 8 | L, L = 2^NB - 1 - off (0 at t >= cap)
    const uint32_t *pack;
    void *sig;
    unsigned long long *n_sat;
    unsigned long long *item_ctr;
};

// The draw word of cell r for NB stored planes.  CLAMP (planes of min(x, 2^NB - 1),
// the largest bound < 2^(NB + 1)): a draw with off >= 2^NB - 1 cannot be tested
// on the planes; it is flagged (bit 7) with off - (2^NB - 1) in bits 0..6 and
// tested on the rows' bytes in global memory (rare: only the top cells of the
// few columns whose bound exceeds 2^NB - 1).
template <int NB, bool CLAMP = false>
__device__ __forceinline__ uint32_t bs_word(uint32_t r, const uint32_t *pack, uint32_t uni_m, uint32_t GN, uint32_t t,
                                            uint32_t cap) {
    const uint2 d = unpack_cell(cell_of(r, pack, uni_m));
    constexpr uint32_t TOP = (1u << NB) - 1u;
    if (CLAMP && t < cap && d.y >= TOP) return ((d.x * GN) << 8) | 0x80u | (d.y - TOP);
    return ((d.x * GN) << 8) | (t < cap ? TOP - d.y : 0u);
}

template <int NB, bool CLAMP>
__global__ void bs_table_kernel(uint32_t *__restrict__ table, uint32_t k, uint64_t S, uint32_t M,
                                const uint32_t *__restrict__ pack, uint32_t uni_m, uint32_t GN, uint32_t cap) {
    const int64_t total = (int64_t)k * T0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t j = (uint32_t)(i / T0), t = (uint32_t)(i % T0);
        table[i] = bs_word<NB, CLAMP>(draw_r(S, j, t, M), pack, uni_m, GN, t, cap);
    }
}

__device__ __forceinline__ uint32_t prmt_b(uint32_t a, uint32_t b, uint32_t sel) {
    uint32_t d;
    asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(sel));
    return d;
}

__device__ __forceinline__ uint32_t bs_prmt(uint32_t a, uint32_t sel) {
    uint32_t d;
    asm("prmt.b32 %0, %1, 0, %2;" : "=r"(d) : "r"(a), "r"(sel));
    return d;
}

// the NB plane words of (column, group) for the draw word w; blocks of NBS
// words.  With NBS = 8 the two 16-byte halves are loaded in the order of the
// lane's part parity, so the two parts of an 8-lane shared-memory phase (4
// groups each) touch complementary bank quarters: conflict-free for any columns.
template <int NB, int NBS>
__device__ __forceinline__ void bs_load(const uint32_t *pl, uint32_t w, uint32_t h, uint32_t (&x)[NB]) {
    const uint32_t *pp = pl + (w >> 8);
    if (NBS == 8) {
        const uint4 a = reinterpret_cast<const uint4 *>(pp)[h], b = reinterpret_cast<const uint4 *>(pp)[h ^ 1u];
        const uint4 lo = h ? b : a, hi = h ? a : b;
        const uint32_t v[8] = {lo.x, lo.y, lo.z, lo.w, hi.x, hi.y, hi.z, hi.w};
#pragma unroll
        for (int i = 0; i < NB; i++) x[i] = v[i];
    } else if (NBS == 4) {
        const uint4 a = *reinterpret_cast<const uint4 *>(pp);
        const uint32_t v[4] = {a.x, a.y, a.z, a.w};
#pragma unroll
        for (int i = 0; i < NB; i++) x[i] = v[i];
    } else if (NBS % 2 == 0) {
#pragma unroll
        for (int i = 0; i < NB / 2; i++) {
            const uint2 v = reinterpret_cast<const uint2 *>(pp)[i];
            x[2 * i] = v.x; x[2 * i + 1] = v.y;
        }
    } else {
#pragma unroll
        for (int i = 0; i < NB; i++) x[i] = pp[i];
    }
}

// green mask of the 32 rows (planes x) for the draw word w: the carry out of x + L
template <int NB>
__device__ __forceinline__ uint32_t bs_test(const uint32_t (&x)[NB], uint32_t w) {
    const uint32_t L = w & 0xFFu;
    // L * (1 + 2^9 + 2^18 + 2^27) puts L's bits 7, 6, 5, 4 at the byte MSBs 7, 15, 23, 31
    // (the four copies do not overlap), L * 2^4 * (...) bits 3, 2, 1, 0
    const uint32_t Xh = L * 0x08040201u, Xl = L * 0x80402010u;
    uint32_t c = 0;
#pragma unroll
    for (int b = 0; b < NB; b++) {
        const uint32_t m = bs_prmt(b < 4 ? Xl : Xh, 0x8888u + 0x1111u * (uint32_t)(3 - (b & 3)));
        c = b == 0 ? (x[0] & m) : ((x[b] & m) | (x[b] & c) | (m & c));
    }
    return c;
}

// 8x8 bit transpose of (hi:lo), byte i = row i -> byte b = bit b of rows 0..7
__device__ __forceinline__ void bs_t8(uint32_t &lo, uint32_t &hi) {
    uint32_t t;
    t = (lo ^ (lo >> 7)) & 0x00AA00AAu; lo ^= t ^ (t << 7);
    t = (hi ^ (hi >> 7)) & 0x00AA00AAu; hi ^= t ^ (t << 7);
    t = (lo ^ (lo >> 14)) & 0x0000CCCCu; lo ^= t ^ (t << 14);
    t = (hi ^ (hi >> 14)) & 0x0000CCCCu; hi ^= t ^ (t << 14);
    t = (lo ^ (hi << 4)) & 0xF0F0F0F0u; lo ^= t; hi ^= t >> 4;
}

template <int NB, bool CLAMP>
__device__ __forceinline__ uint32_t bs_late(const BsParams &p, uint64_t keyj, uint32_t t, uint32_t GN) {
    return bs_word<NB, CLAMP>(mulhi_range(splitmix64(keyj ^ (uint64_t)t), p.M), p.pack, p.uni_m, GN, t, p.cap);
}

// a flagged draw (CLAMP): x[row][c] > off read from the rows themselves
template <int NB>
__device__ __noinline__ uint32_t bs_slow(const BsParams &p, int64_t grow0, int nrg, uint32_t w, uint32_t GN) {
    const uint32_t c = (w >> 8) / GN, off = (1u << NB) - 1u + (w & 0x7Fu);
    const uint8_t *xc = p.x + grow0 * (int64_t)p.D + c;
    uint32_t m = 0;
    for (int i = 0; i < nrg; i++) m |= (uint32_t)(__ldg(xc + (int64_t)i * p.D) > off) << i;
    return m;
}

template <int NB, int NBS, int G, bool CLAMP = false>
__global__ void __launch_bounds__(BS_NT, 1) hash_tiled_bs_kernel(const BsParams p) {
    // rows, lanes per group, draws per lane per round, draws per group per round
    constexpr int R = 32 * G, LP = 32 / G, DPL = bs_dpl(G), RD = LP * DPL;
    static_assert(DPL <= 16, "the record loop decodes 4 bits of draw index");
    extern __shared__ __align__(16) uint32_t smem[];
    // SPLIT (unpadded NB = 5..7): planes 0..3 of (column, group) as one 16-byte
    // block [D][G][4], the other NB - 4 in a second array [D][G][NB - 4]: two
    // shared loads per draw instead of three or more
    constexpr bool SPLIT = NBS == NB && NB > 4 && NB < 8;
    uint32_t *planes = smem;                                                       // [D][G][NBS] (or split)
    const size_t pl_words = ((size_t)p.D * G * NBS + 3) & ~(size_t)3;
    uint32_t *planesB = planes + (size_t)p.D * G * 4;                              // SPLIT: [D][G][NB - 4]
    uint32_t *sbuf_all = planes + pl_words;                                        // [NW][T0]
    uint16_t *hres_all = reinterpret_cast<uint16_t *>(sbuf_all + BS_NW * T0);     // [NW][HB][R]
    __shared__ long long s_item, s_next;
    __shared__ int s_hash;
    __shared__ uint32_t s_live[G];

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t *sbuf = sbuf_all + warp * T0;
    uint16_t *hres_blk = hres_all + warp * BS_HB * R;
    unsigned long long sat = 0;
    const int quads = p.D >> 2;                        // D % 4 == 0 (launcher)
    uint8_t *pbytes = reinterpret_cast<uint8_t *>(planes);
    if (threadIdx.x == 0) s_next = (long long)atomicAdd(p.item_ctr, 1ull);

    for (;;) {
        __syncthreads();
        if (threadIdx.x == 0) {
            s_item = s_next;
            s_next = (long long)atomicAdd(p.item_ctr, 1ull);
            s_hash = 0;
        }
        if (threadIdx.x < G) s_live[threadIdx.x] = 0;
        __syncthreads();
        const long long item = s_item;
        if (item >= p.n_items) break;
        if (s_next < p.n_items) {                      // warm L2 with the next item's rows
            const int64_t nrow0 = (s_next / p.n_hchunks) * R;
            const int64_t nbytes = min((int64_t)R, p.n_rows - nrow0) * (int64_t)p.D;
            const char *base = reinterpret_cast<const char *>(p.x + nrow0 * (int64_t)p.D);
            for (int64_t off = (int64_t)threadIdx.x * 128; off < nbytes; off += (int64_t)BS_NT * 128)
                asm volatile("prefetch.global.L2 [%0];" ::"l"(base + off));
        }
        const int64_t tile = item / p.n_hchunks;
        const int hc = (int)(item % p.n_hchunks);
        const int64_t row0 = tile * R;
        const int nr = (int)min((int64_t)R, p.n_rows - row0);
        const uint32_t j0 = (uint32_t)hc * p.hchunk, j1 = min(p.k, j0 + (uint32_t)p.hchunk);

        // ---- a5: stage as bit planes.  Unit = (column quad, group, octet of 8
        //      rows), octet fastest; 8 words in, 4 columns x NB plane bytes out
        for (int u = threadIdx.x; u < quads * G * 4; u += BS_NT) {
            const int o = u & 3, g = (u >> 2) % G, cq = (u >> 2) / G;
            const int rb = 32 * g + 8 * o;
            uint32_t w[8];
            uint32_t live = 0;
#pragma unroll
            for (int i = 0; i < 8; i++) {
                const bool ok = rb + i < nr;
                w[i] = ok ? __ldg(reinterpret_cast<const uint32_t *>(p.x + (row0 + rb + i) * (int64_t)p.D) + cq) : 0u;
                live |= (w[i] != 0u) << i;
                if (CLAMP) w[i] = __vminu4(w[i], ((1u << NB) - 1u) * 0x01010101u);
            }
            if (live) atomicOr(&s_live[g], live << (8 * o));
            // 4x4 byte transposes: col[u4] = byte u4 of rows 0..3 (lo) and 4..7 (hi)
            uint32_t lo[4], hi[4];
            {
                const uint32_t t0 = prmt_b(w[0], w[1], 0x5140), t1 = prmt_b(w[0], w[1], 0x7362);
                const uint32_t t2 = prmt_b(w[2], w[3], 0x5140), t3 = prmt_b(w[2], w[3], 0x7362);
                lo[0] = prmt_b(t0, t2, 0x5410); lo[1] = prmt_b(t0, t2, 0x7632);
                lo[2] = prmt_b(t1, t3, 0x5410); lo[3] = prmt_b(t1, t3, 0x7632);
                const uint32_t s0 = prmt_b(w[4], w[5], 0x5140), s1 = prmt_b(w[4], w[5], 0x7362);
                const uint32_t s2 = prmt_b(w[6], w[7], 0x5140), s3 = prmt_b(w[6], w[7], 0x7362);
                hi[0] = prmt_b(s0, s2, 0x5410); hi[1] = prmt_b(s0, s2, 0x7632);
                hi[2] = prmt_b(s1, s3, 0x5410); hi[3] = prmt_b(s1, s3, 0x7632);
            }
#pragma unroll
            for (int u4 = 0; u4 < 4; u4++) {
                uint32_t a = lo[u4], b = hi[u4];
                bs_t8(a, b);
                const size_t blk = (size_t)(4 * cq + u4) * G + g;
                if (SPLIT) {
                    uint8_t *dA = pbytes + blk * 16 + o;
                    uint8_t *dB = reinterpret_cast<uint8_t *>(planesB) + blk * (NB - 4) * 4 + o;
#pragma unroll
                    for (int pb = 0; pb < NB; pb++) {
                        const uint8_t v = (uint8_t)((pb < 4 ? a : b) >> (8 * (pb & 3)));
                        if (pb < 4) dA[4 * pb] = v;
                        else dB[4 * (pb - 4)] = v;
                    }
                } else {
                    uint8_t *dst = pbytes + blk * NBS * 4 + o;
#pragma unroll
                    for (int pb = 0; pb < NB; pb++) dst[4 * pb] = (uint8_t)((pb < 4 ? a : b) >> (8 * (pb & 3)));
                }
            }
        }
        __syncthreads();

        // ---- hashes: a warp claims blocks of BS_HB consecutive hashes (the next
        //      block one block ahead), prefetches the next hash's draws, and
        //      flushes a block's results with one store per row ------------------
        auto grab = [&]() {
            int bb = 0;
            if (lane == 0) bb = atomicAdd(&s_hash, 1);
            return min(j1, j0 + (uint32_t)BS_HB * (uint32_t)__shfl_sync(0xFFFFFFFFu, bb, 0));
        };
        const int g = lane % G, part = lane / G;          // groups fastest: the G lanes of a part share a column
        const uint32_t *plg = planes + g * NBS;
        const uint32_t GN = (uint32_t)(SPLIT ? G : G * NBS);   // the table's column stride
        const uint32_t live0 = s_live[g];
        const uint32_t valid = 32 * g + 32 <= nr ? 0xFFFFFFFFu : (32 * g >= nr ? 0u : (1u << (nr - 32 * g)) - 1u);
        const uint32_t pend0 = live0 & valid;
        const uint32_t dead = valid & ~live0;
        uint32_t jb = grab();                          // current block [jb, je)
        uint32_t je = min(j1, jb + BS_HB);
        uint32_t jb_next = jb < j1 ? grab() : j1;
        uint32_t j = jb;
        uint4 pre[2];                                  // T0 = 256 draws = 2 x 16 B per lane
        if (j < j1) {
            const uint4 *t4 = reinterpret_cast<const uint4 *>(p.table + (int64_t)j * T0);
            pre[0] = __ldg(t4 + lane);
            pre[1] = __ldg(t4 + 32 + lane);
        }
        while (j < j1) {
            __syncwarp();
            reinterpret_cast<uint4 *>(sbuf)[lane] = pre[0];
            reinterpret_cast<uint4 *>(sbuf)[32 + lane] = pre[1];
            __syncwarp();
            const uint32_t jn = j + 1 < je ? j + 1 : jb_next;
            uint16_t *hres = hres_blk + (j - jb) * R;
            if (jn < j1) {
                const uint4 *t4 = reinterpret_cast<const uint4 *>(p.table + (int64_t)jn * T0);
                pre[0] = __ldg(t4 + lane);
                pre[1] = __ldg(t4 + 32 + lane);
            }
            const uint64_t keyj = p.S ^ ((uint64_t)j << 32);
            // all-zero rows: cap at once (part 0 of each group writes them)
            if (part == 0 && dead) {
                uint32_t d = dead;
                while (d) {
                    const int b = __ffs(d) - 1;
                    hres[32 * g + b] = (uint16_t)p.cap;
                    d &= d - 1;
                }
                sat += __popc(dead);
            }
            uint32_t pend = pend0;
            for (uint32_t tb = 0;; tb += RD) {
                if (!__any_sync(0xFFFFFFFFu, pend != 0u)) break;
                if (tb >= p.cap) {                     // a9: no green draw before the cap
                    if (part == 0) {
                        uint32_t d = pend;
                        while (d) {
                            const int b = __ffs(d) - 1;
                            hres[32 * g + b] = (uint16_t)p.cap;
                            d &= d - 1;
                        }
                        sat += __popc(pend);
                    }
                    break;
                }
                const uint32_t t0 = tb + (uint32_t)(part * DPL);
                // all DPL draw words, then all plane loads, then the tests (loads in flight together)
                uint32_t wd[DPL];
                if (tb + RD <= (uint32_t)T0) {
#pragma unroll
                    for (int i = 0; i < DPL; i++) wd[i] = sbuf[t0 + i];
                } else {
#pragma unroll
                    for (int i = 0; i < DPL; i++)
                        wd[i] = t0 + i < (uint32_t)T0 ? sbuf[t0 + i] : bs_late<NB, CLAMP>(p, keyj, t0 + i, GN);
                }
                uint32_t xv[DPL][NB];
#pragma unroll
                for (int i = 0; i < DPL; i++) {
                    if constexpr (SPLIT) {
                        const uint32_t blk = (wd[i] >> 8) + (uint32_t)g;              // (column, group) block
                        const uint4 a4 = reinterpret_cast<const uint4 *>(planes)[blk];
                        xv[i][0] = a4.x; xv[i][1] = a4.y; xv[i][2] = a4.z; xv[i][3] = a4.w;
                        const uint32_t *pb = planesB + blk * (NB - 4);
                        if (NB - 4 == 2) {
                            const uint2 b2 = *reinterpret_cast<const uint2 *>(pb);
                            xv[i][4 % NB] = b2.x; xv[i][5 % NB] = b2.y;
                        } else {
#pragma unroll
                            for (int q = 4; q < NB; q++) xv[i][q] = pb[q - 4];
                        }
                    } else {
                        bs_load<NB, NBS>(plg, wd[i], (uint32_t)part & 1u, xv[i]);
                    }
                }
                uint32_t gms[DPL];
#pragma unroll
                for (int i = 0; i < DPL; i++) gms[i] = bs_test<NB>(xv[i], wd[i]);
                if (CLAMP) {                         // one test for the lane's DPL draws, then the rare ones
                    uint32_t fl = 0;
#pragma unroll
                    for (int i = 0; i < DPL; i++) fl |= wd[i];
                    if (fl & 0x80u) {
#pragma unroll
                        for (int i = 0; i < DPL; i++)
                            if (wd[i] & 0x80u) gms[i] = bs_slow<NB>(p, row0 + 32 * g, min(32, nr - 32 * g), wd[i], GN);
                    }
                }
                uint32_t F[DPL], any = 0;
#pragma unroll
                for (int i = 0; i < DPL; i++) {
                    F[i] = gms[i] & ~any;
                    any |= gms[i];
                }
                // segmented prefix OR over the group's parts (lanes g, g + G, ...; draw order = part order)
                uint32_t incl = any;
#pragma unroll
                for (int o = 1; o < LP; o <<= 1) {
                    const uint32_t v = __shfl_up_sync(0xFFFFFFFFu, incl, o * G);
                    if (part >= o) incl |= v;
                }
                uint32_t excl = __shfl_up_sync(0xFFFFFFFFu, incl, G);
                if (part == 0) excl = 0;
                // rows first green in this lane's draws: one loop over all of them,
                // the draw index i from its bits (the F[i] are disjoint)
                uint32_t n = any & ~excl & pend;
                uint32_t B0 = 0, B1 = 0, B2 = 0, B3 = 0;
#pragma unroll
                for (int i = 1; i < DPL; i++) {
                    if (i & 1) B0 |= F[i];
                    if (i & 2) B1 |= F[i];
                    if (i & 4) B2 |= F[i];
                    if (i & 8) B3 |= F[i];
                }
                while (n) {
                    const int b = __ffs(n) - 1;
                    const uint32_t i = ((B0 >> b) & 1u) | (((B1 >> b) & 1u) << 1) | (((B2 >> b) & 1u) << 2) |
                                       (((B3 >> b) & 1u) << 3);
                    hres[32 * g + b] = (uint16_t)(t0 + i + 1);
                    n &= n - 1;
                }
                pend &= ~__shfl_sync(0xFFFFFFFFu, incl, (LP - 1) * G + g);
            }
            __syncwarp();
            if (j + 1 == je) {
                // ---- a9: flush the block: row r's hashes jb..je-1 are contiguous in sig
                const int64_t eoff = (row0 + lane) * (int64_t)p.k + jb;
                const int nh = (int)(je - jb);
                if (nh == BS_HB && p.vec_flush) {
                    for (int r = lane; r < nr; r += 32) {
                        const int64_t e = eoff + (int64_t)(r - lane) * p.k;
                        uint32_t hv[BS_HB];
#pragma unroll
                        for (int u = 0; u < BS_HB; u++) hv[u] = hres_blk[u * R + r];
                        if (p.sigb == 2) {
                            uint16_t *ptr = reinterpret_cast<uint16_t *>(p.sig) + e;
                            const uint4 v = make_uint4(hv[0] | (hv[1] << 16), hv[2] | (hv[3] << 16),
                                                       hv[4] | (hv[5] << 16), hv[6] | (hv[7] << 16));
                            if (p.vec_flush == 2) {
                                *reinterpret_cast<uint4 *>(ptr) = v;
                            } else {
                                reinterpret_cast<uint2 *>(ptr)[0] = make_uint2(v.x, v.y);
                                reinterpret_cast<uint2 *>(ptr)[1] = make_uint2(v.z, v.w);
                            }
                        } else {
                            uint8_t *ptr = reinterpret_cast<uint8_t *>(p.sig) + e;
                            *reinterpret_cast<uint2 *>(ptr) = make_uint2(hv[0] | (hv[1] << 8) | (hv[2] << 16) | (hv[3] << 24),
                                                                         hv[4] | (hv[5] << 8) | (hv[6] << 16) | (hv[7] << 24));
                        }
                    }
                } else {
                    for (int r = lane; r < nr; r += 32) {
                        const int64_t e = eoff + (int64_t)(r - lane) * p.k;
                        for (int u = 0; u < nh; u++) {
                            if (p.sigb == 2) reinterpret_cast<uint16_t *>(p.sig)[e + u] = hres_blk[u * R + r];
                            else reinterpret_cast<uint8_t *>(p.sig)[e + u] = (uint8_t)hres_blk[u * R + r];
                        }
                    }
                }
                __syncwarp();
                jb = jb_next;
                je = min(j1, jb + BS_HB);
                jb_next = jb < j1 ? grab() : j1;
            }
            j = jn;
        }
    }
    if (p.n_sat) {
        for (int o = 16; o; o >>= 1) sat += __shfl_xor_sync(0xFFFFFFFFu, sat, o);
        if (lane == 0 && sat) atomicAdd(p.n_sat, sat);
    }
}

static size_t bs_smem(int D, int G, int NBS) {
    return (((size_t)D * G * NBS + 3) & ~(size_t)3) * 4 + (size_t)BS_NW * T0 * 4 + (size_t)BS_NW * BS_HB * 32 * G * 2;
}

template <int NB, int NBS, int G, bool CLAMP = false>
static void bs_launch(const BsParams &p, size_t smem, int grid, cudaStream_t s) {
    auto kern = hash_tiled_bs_kernel<NB, NBS, G, CLAMP>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kernel_timer_begin(s);
    kern<<<grid, BS_NT, smem, s>>>(p);
    kernel_timer_end(s);
}

// (NBS, G): padded blocks of 4 words with 8 groups or 8 words with 4 groups are
// bank-conflict-free (an 8-lane phase covers 32 distinct banks); smaller G
// (long rows) and unpadded blocks (NBS = NB, 5..7) trade conflicts for space
template <int NB>
static void bs_launch_nb(int NBS, int G, const BsParams &p, size_t smem, int grid, cudaStream_t s) {
    if (NBS == 4) {
        if constexpr (NB <= 4) {
            if (G == 8) bs_launch<NB, 4, 8>(p, smem, grid, s);
            else if (G == 4) bs_launch<NB, 4, 4>(p, smem, grid, s);
            else if (G == 2) bs_launch<NB, 4, 2>(p, smem, grid, s);
            else bs_launch<NB, 4, 1>(p, smem, grid, s);
        }
    } else if (NBS == 8) {
        if constexpr (NB > 4) {
            if (G == 4) bs_launch<NB, 8, 4>(p, smem, grid, s);
            else if (G == 2) bs_launch<NB, 8, 2>(p, smem, grid, s);
            else bs_launch<NB, 8, 1>(p, smem, grid, s);
        }
    } else if (NBS == NB) {
        if constexpr (NB > 4 && NB < 8) {
            if (G == 2) bs_launch<NB, NB, 2>(p, smem, grid, s);
            else bs_launch<NB, NB, 1>(p, smem, grid, s);
        }
    } else {                                     // NBS = -NB: clamped planes, 2 groups
        if constexpr (NB >= 4 && NB < 8) bs_launch<NB, NB, 2, true>(p, smem, grid, s);
    }
}

template <int NB>
static void bs_table(uint32_t *table, const HashArgs &a, uint32_t uni_m, uint32_t GN, bool clamp, cudaStream_t s) {
    const int64_t total = (int64_t)a.k * T0;
    const int blocks = (int)min((int64_t)num_sms() * 8, (total + 255) / 256);
    if (clamp) bs_table_kernel<NB, true><<<blocks, 256, 0, s>>>(table, a.k, a.S, (uint32_t)a.L->M, a.L->cell_pack, uni_m, GN, a.cap);
    else bs_table_kernel<NB, false><<<blocks, 256, 0, s>>>(table, a.k, a.S, (uint32_t)a.L->M, a.L->cell_pack, uni_m, GN, a.cap);
}

#define WMH_BS_NB_SWITCH(NBV, CALL) \
    switch (NBV) {                  \
        case 1: CALL(1); break;     \
        case 2: CALL(2); break;     \
        case 3: CALL(3); break;     \
        case 4: CALL(4); break;     \
        case 5: CALL(5); break;     \
        case 6: CALL(6); break;     \
        case 7: CALL(7); break;     \
        default: CALL(8); break;    \
    }

wmh_status launch_hash_tiled_bs(const HashArgs &a, bool *handled) {
    *handled = false;
    const int D = (int)a.rows.dim;
    if (a.rows.kind != WMH_DENSE || (D & 3) || ((uintptr_t)a.rows.dense & 3)) return WMH_OK;
    if ((a.L->flags & WMH_LAYOUT_WIDE) || a.L->max_bound == 0 || a.L->max_bound > 255) return WMH_OK;
    const int NB = 32 - __builtin_clz(a.L->max_bound);
    int dev = 0;
    cudaGetDevice(&dev);
    int smem_optin = 0;
    cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    static const int g_env = getenv("WMH_BS_GROUPS") ? atoi(getenv("WMH_BS_GROUPS")) : 0;
    // padded (conflict-free) first, then fewer groups, then unpadded blocks
    int NBS = NB <= 4 ? 4 : 8, G = NB <= 4 ? 8 : 4;
    if (g_env > 0 && g_env <= G && (g_env & (g_env - 1)) == 0) G = g_env;
    while (G >= 1 && bs_smem(D, G, NBS) > (size_t)smem_optin) G /= 2;
    if (G < 2 && NB > 4 && NB < 8 && bs_smem(D, 2, NB) <= (size_t)smem_optin) { NBS = NB; G = 2; }
    // still one group: NB - 1 planes of min(x, 2^(NB-1) - 1) when the draws they
    // cannot decide (the top cells of the columns with m_c >= 2^(NB-1)) are rare
    int NBP = NB;                                // planes stored and tested
    bool clamp = false;
    if (G < 2 && NB >= 5 && bs_smem(D, 2, NB - 1) <= (size_t)smem_optin) {
        // cells above the clamp, counted once by wmh_prepare (no device round trip here)
        const uint64_t flagged = a.L->clamp_cells[NB - 1];
        static const double max_frac = getenv("WMH_BS_CLAMP_FRAC") ? atof(getenv("WMH_BS_CLAMP_FRAC")) : 1e-3;
        if ((double)flagged <= max_frac * (double)a.L->M) { NBP = NB - 1; NBS = -NBP; G = 2; clamp = true; }
    }
    if (G < 1 && NB > 4 && NB < 8 && bs_smem(D, 1, NB) <= (size_t)smem_optin) { NBS = NB; G = 1; }
    if (G < 1) return WMH_OK;
    // auto choice: a one-group tile (32 rows, one draw per lane per round) loses
    // to the byte tile (c5 at full size, NB = 7: 498 vs 377 ms)
    if (a.tile != 2 && G < 2) return WMH_OK;
    const int NBSW = NBS < 0 ? -NBS : NBS;        // words per (column, group) block
    if ((uint64_t)D * G * NBSW >= (1ull << 23)) return WMH_OK;
    const size_t smem = bs_smem(D, G, NBSW);
    const int R = 32 * G;
    *handled = true;

    const int64_t n_tiles = (a.rows.n_rows + R - 1) / R;
    const int sms = num_sms();
    // >= 8 items per SM for balance, but >= WMH_MIN_HCHUNK hashes per item: each
    // item stages its whole tile, so small batches must not slice k too thin
    // (a 3,300-row batch of c2 in 16-hash items ran 3x slower than its share)
    static const int min_hc = getenv("WMH_MIN_HCHUNK") ? std::max(8, atoi(getenv("WMH_MIN_HCHUNK"))) : 128;
    int n_hchunks = (int)max((int64_t)1, min((int64_t)(a.k + min_hc - 1) / min_hc, ((int64_t)sms * 8 + n_tiles - 1) / n_tiles));
    static const int hc_env = getenv("WMH_CM_HCHUNKS") ? atoi(getenv("WMH_CM_HCHUNKS")) : 0;
    if (hc_env > 0) n_hchunks = (int)min((int64_t)hc_env, (int64_t)(a.k + BS_HB - 1) / BS_HB);
    const int hchunk = (int)(((a.k + n_hchunks - 1) / n_hchunks + BS_HB - 1) / BS_HB * BS_HB);
    n_hchunks = (int)((a.k + hchunk - 1) / hchunk);

    uint8_t *scratch = nullptr;
    const size_t tab_bytes = (size_t)a.k * T0 * sizeof(uint32_t);
    WMH_CUDA_TRY(cudaMallocAsync((void **)&scratch, tab_bytes + 256, a.stream), "tiled scratch alloc");
    uint32_t *table = reinterpret_cast<uint32_t *>(scratch);
    unsigned long long *ctr = reinterpret_cast<unsigned long long *>(scratch + tab_bytes);
    WMH_CUDA_TRY(cudaMemsetAsync(ctr, 0, sizeof(unsigned long long), a.stream), "tiled counter memset");
    const uint32_t uni_m = (a.L->flags & WMH_LAYOUT_UNIFORM) ? a.L->uniform_m : 0u;
    // column stride of the draw words: (column, group) blocks for the split
    // layout of unpadded 5..7 planes (the kernel's SPLIT), else words
    const bool split = NBSW == NBP && NBP > 4 && NBP < 8;
    const uint32_t GN = (uint32_t)(split ? G : G * NBSW);
#define WMH_BS_TAB(V) bs_table<V>(table, a, uni_m, GN, clamp, a.stream)
    WMH_BS_NB_SWITCH(NBP, WMH_BS_TAB)
#undef WMH_BS_TAB
    count_launch();
    if (cudaGetLastError() != cudaSuccess) { cudaFreeAsync(scratch, a.stream); return cuda_fail(cudaGetLastError(), "bs table launch"); }

    BsParams p;
    p.x = a.rows.dense;
    p.n_rows = a.rows.n_rows;
    p.D = D;
    p.G = G;
    p.n_hchunks = n_hchunks;
    p.hchunk = hchunk;
    p.n_items = n_tiles * n_hchunks;
    p.k = a.k;
    p.cap = a.cap;
    p.M = (uint32_t)a.L->M;
    p.uni_m = uni_m;
    p.S = a.S;
    p.sigb = a.sig_bytes;
    p.vec_flush = 0;
    if (a.sig_bytes == 2 && a.k % 4 == 0 && (uintptr_t)a.sig % 8 == 0)
        p.vec_flush = (a.k % 8 == 0 && (uintptr_t)a.sig % 16 == 0) ? 2 : 1;
    if (a.sig_bytes == 1 && a.k % 8 == 0 && (uintptr_t)a.sig % 8 == 0) p.vec_flush = 1;
    p.table = table;
    p.pack = a.L->cell_pack;
    p.sig = a.sig;
    p.n_sat = a.n_sat;
    p.item_ctr = ctr;
    const int grid = (int)min((int64_t)sms, p.n_items);
#define WMH_BS_GO(V) bs_launch_nb<V>(NBS, G, p, smem, grid, a.stream)
    WMH_BS_NB_SWITCH(NBP, WMH_BS_GO)
#undef WMH_BS_GO
    WMH_LAUNCH_CHECK("hash_tiled_bs launch");
    if (getenv("WMH_TILED_STATS"))
        fprintf(stderr, "[wmh tiled bs] NB=%d planes=%d NBS=%d G=%d grid=%d items=%lld hchunk=%d smem=%zu\n", NB, NBP, NBS, G, grid,
                (long long)p.n_items, hchunk, smem);
    cudaFreeAsync(scratch, a.stream);
    return WMH_OK;
}

}  // namespace wmh
