// hash_bitslice.cu -- WMH_ALGO_TILED for dense uint8 rows: the bit-sliced tile,
// lane = draw.
//
// Same draws, same result as every other kernel (the draw stream of hash j does
// not depend on x, so one draw serves every row of a tile).  A CTA
// stages R = 32*G rows as bit planes: for column c and a group g of 32 rows, P
// words whose bit i is bit b of min(x[32g + i][c], 2^P - 1).  Alg. 5's test of
// one draw (c, off) against the 32 rows of a group is the carry out of the
// bit-serial sum x + L with L = 2^P - 1 - off:
//
//   green(x) <=> x > off <=> x + L >= 2^P,   carry_{b+1} = MAJ(x_b, L_b, carry_b)
//
// one LOP3 per plane for 32 rows (reading R2: strict, integer cells).
//
// Work of a warp per hash, in rounds of BV_RD = 96 draws (Alg. 3's loop,
// P:166-176, unrolled over lanes):
//   screen: lane l decodes draws t = tb + 32 s + l (s < 3; column c, offset off)
//     from the per-launch draw table and compares off with the tile's column
//     maxima gmax[c][g] (kept next to the planes).  A draw can turn a row of group
//     g green only when off < gmax[c][g]; for c5 that is ~25% of the draws.  The
//     needed draws are compacted, in draw order, into a per-warp list (ballot +
//     popcount positions).
//   test: 32 listed draws at a time, lane = draw: build the L_b masks, load the
//     column's plane block, one carry chain per group -> a green mask per group
//     (lane = draw, bit = row).
//   combine: a 32x32 bit transpose per group gives lane = row the list positions
//     with a green; the first one (__ffs) is the row's first green draw, h = t + 1
//     (reading R1).  Rows found leave the pending masks.
// A row stays pending until it is green or the cap is reached (h = cap, R9);
// all-zero rows never turn green and take the cap at once (R12).  A block of 8
// hashes' results is kept in registers (lane = row, two 16-bit h per word) and
// flushed with one 16-byte store per row.
//
// Clamped planes (CLAMP): when the bit count NB of the largest bound would not
// let two groups fit, P = NB - 1 planes hold min(x, 2^P - 1) and gmax the true
// maximum.  A draw with off >= 2^P - 1 is green only for rows whose clamped value
// is all ones; when gmax says such a row exists (rare: the top cells of the few
// columns with a large bound), those candidate rows are tested on their bytes
// in global memory.
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>
#include <cmath>

#include "common.cuh"

namespace wmh {

constexpr int BV_HB = 8;                  // hashes per claimed block (results flushed 8 per row)
constexpr int BV_SB = 1;                  // staging units (quad pairs) per thread whose loads are in flight together
#ifndef WMH_BV_DPL
#define WMH_BV_DPL 3
#endif
#ifndef WMH_BV_NT
#define WMH_BV_NT 640
#endif
constexpr int BV_DPL = WMH_BV_DPL;        // draws screened per lane per round
constexpr int BV_RD = 32 * BV_DPL;        // draws per round
constexpr int BV_T0 = 4 * BV_RD;          // draws per hash kept in the per-launch table (whole rounds)
constexpr int BV_NT = WMH_BV_NT;               // threads per CTA: 20 warps at <= 96 registers (measured on c5: 512 10.59 ms, 640 10.14, 768 14.07 (spills))

struct BvParams {
    const uint8_t *x;
    int64_t n_rows;
    int D;
    int n_hchunks, hchunk;
    int64_t n_items;
    uint32_t k, cap, M, uni_m;
    uint64_t S;
    int vec_flush, sigb;
    const uint32_t *table;       // [k][BV_T0] draw words (c << 8) | off; 0xFF (never green) at t >= cap
    const uint32_t *pack;
    void *sig;
    unsigned long long *n_sat;
    unsigned long long *item_ctr;
    int bulk_pf;                 // rows 16-byte aligned: the next tile's L2 prefetch by TMA bulk prefetches
};

// the draw word of cell r: (c << 8) | (r - CompToM[c]); t >= cap -> 0xFF, which
// no group maximum exceeds (bounds <= 255), so the draw is red everywhere
__device__ __forceinline__ uint32_t bv_word(uint32_t r, const uint32_t *pack, uint32_t uni_m, uint32_t t, uint32_t cap) {
    return t < cap ? cell_of(r, pack, uni_m) : 0xFFu;
}

// the first BV_T0 draw words of every hash; cells by the packed IntToComp table or
// (c2m != null, WMH_OPT_ISGREEN_BINSEARCH) by binary search over CompToM
__global__ void bv_table_kernel(uint32_t *__restrict__ table, uint32_t k, uint64_t S, uint32_t M,
                                const uint32_t *__restrict__ pack, uint32_t uni_m, uint32_t cap,
                                const uint32_t *__restrict__ c2m, uint32_t D) {
    const int64_t total = (int64_t)k * BV_T0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t j = (uint32_t)(i / BV_T0), t = (uint32_t)(i % BV_T0);
        const uint32_t r = draw_r(S, j, t, M);
        if (c2m) {
            const uint2 cell = cell_bsearch(r, c2m, D);
            table[i] = t < cap ? (cell.x << 8) | cell.y : 0xFFu;
        } else {
            table[i] = bv_word(r, pack, uni_m, t, cap);
        }
    }
}

__device__ __forceinline__ uint32_t bv_prmt(uint32_t a, uint32_t b, uint32_t sel) {
    uint32_t d;
    asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(sel));
    return d;
}

__device__ __forceinline__ uint32_t bv_rotl(uint32_t y, uint32_t n) {
    uint32_t d;
    asm("shf.l.wrap.b32 %0, %1, %1, %2;" : "=r"(d) : "r"(y), "r"(n));
    return d;
}

// Per-lane constants of the 32x32 bit transpose (lane i holds row i of the
// matrix; afterwards lane r holds column r).  Stage s swaps the off-diagonal
// s x s blocks between lanes i and i ^ s: lanes with bit s clear keep their bits
// r with r & s == 0 and take the partner's bits shifted up by s; the others keep
// r & s != 0 and take the partner's bits shifted down.  Stages 16 and 8 move
// whole bytes (one PRMT), stages 4, 2, 1 a rotate plus a select (LOP3).
struct BvTranspose {
    uint32_t sel16, sel8, amt4, keep4, amt2, keep2, amt1, keep1;
    __device__ __forceinline__ explicit BvTranspose(int lane) {
        sel16 = (lane & 16) ? 0x3276u : 0x5410u;
        sel8 = (lane & 8) ? 0x3715u : 0x6240u;
        amt4 = (lane & 4) ? 28u : 4u;
        keep4 = (lane & 4) ? 0xF0F0F0F0u : 0x0F0F0F0Fu;
        amt2 = (lane & 2) ? 30u : 2u;
        keep2 = (lane & 2) ? 0xCCCCCCCCu : 0x33333333u;
        amt1 = (lane & 1) ? 31u : 1u;
        keep1 = (lane & 1) ? 0xAAAAAAAAu : 0x55555555u;
    }
    __device__ __forceinline__ uint32_t operator()(uint32_t x) const {
        uint32_t y = __shfl_xor_sync(0xFFFFFFFFu, x, 16);
        x = bv_prmt(x, y, sel16);
        y = __shfl_xor_sync(0xFFFFFFFFu, x, 8);
        x = bv_prmt(x, y, sel8);
        y = __shfl_xor_sync(0xFFFFFFFFu, x, 4);
        x = (x & keep4) | (bv_rotl(y, amt4) & ~keep4);
        y = __shfl_xor_sync(0xFFFFFFFFu, x, 2);
        x = (x & keep2) | (bv_rotl(y, amt2) & ~keep2);
        y = __shfl_xor_sync(0xFFFFFFFFu, x, 1);
        x = (x & keep1) | (bv_rotl(y, amt1) & ~keep1);
        return x;
    }
};

// 8x8 bit transpose of (hi:lo), byte i = row i -> byte b = bit b of rows 0..7
__device__ __forceinline__ void bv_t8(uint32_t &lo, uint32_t &hi) {
    uint32_t t;
    t = (lo ^ (lo >> 7)) & 0x00AA00AAu; lo ^= t ^ (t << 7);
    t = (hi ^ (hi >> 7)) & 0x00AA00AAu; hi ^= t ^ (t << 7);
    t = (lo ^ (lo >> 14)) & 0x0000CCCCu; lo ^= t ^ (t << 14);
    t = (hi ^ (hi >> 14)) & 0x0000CCCCu; hi ^= t ^ (t << 14);
    t = (lo ^ (hi << 4)) & 0xF0F0F0F0u; lo ^= t; hi ^= t >> 4;
}

// bit select: (m & x) | (~m & y), one LOP3 when m is in a register
__device__ __forceinline__ uint32_t bv_sel(uint32_t m, uint32_t x, uint32_t y) {
    uint32_t d;
    asm("lop3.b32 %0, %1, %2, %3, 0xCA;" : "=r"(d) : "r"(m), "r"(x), "r"(y));
    return d;
}

// Delta swap of bit blocks between two row words (one stage of an 8x8 bit
// transpose per byte): bits j of a with j & S != 0 <-> bits j - S of b.  The
// masks m and mh = m << S come in registers (two shifts and two selects).
template <int S>
__device__ __forceinline__ void bv_swap(uint32_t &a, uint32_t &b, uint32_t m, uint32_t mh) {
    const uint32_t x = a >> S, y = b << S;
    b = bv_sel(m, x, b);
    a = bv_sel(mh, y, a);
}

// Column block of the planes: W = G*P words.  P % 4 == 0: group-major [g][b]
// (each group's planes one or two 16-byte loads, loaded only when the group
// needs them); else plane-major [b][g] (the whole block in 16/8/4-byte loads).
template <int P, int G>
struct BvLayout {
    static constexpr int W = G * P;
    static constexpr bool GROUP_MAJOR = P % 4 == 0;
    static __device__ __forceinline__ int idx(int g, int b) { return GROUP_MAJOR ? g * P + b : b * G + g; }
};

// Predicated shared-memory loads at 32-bit shared addresses: when `p` is false
// the registers keep whatever they held (the caller masks those lanes' results).
__device__ __forceinline__ void bv_lds4(uint32_t addr, bool p, uint32_t &a, uint32_t &b, uint32_t &c, uint32_t &d) {
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %5, 0;\n\t@q ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];\n\t}"
                 : "+r"(a), "+r"(b), "+r"(c), "+r"(d) : "r"(addr), "r"((int)p));
}
__device__ __forceinline__ void bv_lds2(uint32_t addr, bool p, uint32_t &a, uint32_t &b) {
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %3, 0;\n\t@q ld.shared.v2.u32 {%0, %1}, [%2];\n\t}"
                 : "+r"(a), "+r"(b) : "r"(addr), "r"((int)p));
}
__device__ __forceinline__ void bv_lds1(uint32_t addr, bool p, uint32_t &a) {
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q ld.shared.u32 %0, [%1];\n\t}"
                 : "+r"(a) : "r"(addr), "r"((int)p));
}

// group g's P plane words of the column block at shared address blk (group-major)
template <int P, int G>
__device__ __forceinline__ void bv_load_group(uint32_t blk, int g, bool p, uint32_t (&x)[P]) {
#pragma unroll
    for (int i = 0; i < P / 4; i++) bv_lds4(blk + 16u * (uint32_t)(g * P / 4 + i), p, x[4 * i], x[4 * i + 1], x[4 * i + 2], x[4 * i + 3]);
}

// the whole column block (W = G*P words) in 16/8/4-byte loads
template <int P, int G>
__device__ __forceinline__ void bv_load_all(uint32_t blk, bool p, uint32_t (&x)[G][P]) {
    constexpr int W = G * P;
    uint32_t v[W];
    if constexpr (W % 4 == 0) {
#pragma unroll
        for (int i = 0; i < W / 4; i++) bv_lds4(blk + 16u * i, p, v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
    } else if constexpr (W % 2 == 0) {
#pragma unroll
        for (int i = 0; i < W / 2; i++) bv_lds2(blk + 8u * i, p, v[2 * i], v[2 * i + 1]);
    } else {
#pragma unroll
        for (int i = 0; i < W; i++) bv_lds1(blk + 4u * i, p, v[i]);
    }
#pragma unroll
    for (int g = 0; g < G; g++)
#pragma unroll
        for (int b = 0; b < P; b++) x[g][b] = v[BvLayout<P, G>::idx(g, b)];
}

// carry out of x + L over the P planes; m[b] = all-ones where bit b of L is set
template <int P>
__device__ __forceinline__ uint32_t bv_chain(const uint32_t (&x)[P], const uint32_t (&m)[P]) {
    uint32_t c = x[0] & m[0];
#pragma unroll
    for (int b = 1; b < P; b++) c = (x[b] & m[b]) | (x[b] & c) | (m[b] & c);
    return c;
}

// group maxima per column: G bytes (G <= 4) in one 1/2/4-byte word
template <int G>
using bv_gmax_t = typename std::conditional<G == 1, uint8_t, typename std::conditional<G == 2, uint16_t, uint32_t>::type>::type;

// CLAMP: the draw (c, off >= 2^P - 1) against the rows of group g whose clamped
// value is all ones (cand), read from the rows in global memory
__device__ __forceinline__ uint32_t bv_slow(const uint8_t *x, int64_t grow0, int D, uint32_t c, uint32_t off, uint32_t cand) {
    uint32_t m = 0;
    while (cand) {
        const int i = __ffs(cand) - 1;
        cand &= cand - 1;
        m |= (uint32_t)(__ldg(x + (grow0 + i) * (int64_t)D + c) > off) << i;
    }
    return m;
}

// Green masks of a listed (needed) draw word w against all G groups; lanes
// without a draw (valid false) load nothing and get empty masks.  CLAMP: true
// when off >= 2^P - 1 (the exact test on the candidate rows follows).
template <int P, int G, bool CLAMP>
__device__ __forceinline__ bool bv_test_c(uint32_t planes_s, uint32_t w, bool valid, uint32_t (&mask)[G]) {
    constexpr uint32_t TOP = (1u << P) - 1u;
    const uint32_t c = w >> 8, off = w & 0xFFu;
    const uint32_t blk = planes_s + c * (uint32_t)(G * P * 4);
    const uint32_t L = CLAMP ? (off < TOP ? TOP - off : 0u) : TOP - off;
    const uint32_t Xh = L * 0x08040201u, Xl = L * 0x80402010u;
    uint32_t m[P];
#pragma unroll
    for (int b = 0; b < P; b++) m[b] = bv_prmt(b < 4 ? Xl : Xh, 0, 0x8888u + 0x1111u * (uint32_t)(3 - (b & 3)));
    if constexpr (BvLayout<P, G>::GROUP_MAJOR) {
#pragma unroll
        for (int g = 0; g < G; g++) {
            uint32_t xg[P];
            bv_load_group<P, G>(blk, g, valid, xg);
            mask[g] = valid ? bv_chain<P>(xg, m) : 0u;
        }
    } else {
        uint32_t xa[G][P];
        bv_load_all<P, G>(blk, valid, xa);
#pragma unroll
        for (int g = 0; g < G; g++) mask[g] = valid ? bv_chain<P>(xa[g], m) : 0u;
    }
    return CLAMP && valid && off >= TOP;
}

// CLAMP, off >= 2^P - 1: the draw against group g's rows whose clamped value
// is all ones, read from the rows in global memory (rare: the top cells of the
// few columns whose bound exceeds 2^P - 1)
template <int P, int G>
__device__ __forceinline__ uint32_t bv_test_slow(const BvParams &p, uint32_t planes_s, const bv_gmax_t<G> *gmax, int64_t row0,
                                              uint32_t w, uint32_t pend, int g) {
    const uint32_t c = w >> 8, off = w & 0xFFu;
    WMH_DASSERT(c < (uint32_t)p.D);
    if (pend == 0u || off >= (((uint32_t)gmax[c] >> (8 * g)) & 0xFFu)) return 0u;
    const uint32_t blk = planes_s + c * (uint32_t)(G * P * 4);
    uint32_t cand = 0xFFFFFFFFu;
    for (int b = 0; b < P; b++) {
        uint32_t v;
        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(blk + 4u * (uint32_t)BvLayout<P, G>::idx(g, b)));
        cand &= v;
    }
    return bv_slow(p.x, row0 + 32 * g, p.D, c, off, cand);
}

template <int P, int G, bool CLAMP, int NT>
__global__ void __launch_bounds__(NT, 1) hash_bitslice_kernel(const BvParams p) {
    constexpr int R = 32 * G;
    constexpr int W = G * P;
    constexpr uint32_t TOP = (1u << P) - 1u;
    using gm_t = bv_gmax_t<G>;
    extern __shared__ __align__(16) uint32_t smem[];
    uint32_t *planes = smem;                                                         // [D][W]
    gm_t *gmax = reinterpret_cast<gm_t *>(planes + (size_t)p.D * W);                 // [D] (G bytes each)
    uint32_t *cbuf_all = reinterpret_cast<uint32_t *>(
        reinterpret_cast<uint8_t *>(gmax) + (((size_t)p.D * sizeof(gm_t) + 15) & ~(size_t)15));   // [NW][BV_RD]
    uint8_t *gbytes = reinterpret_cast<uint8_t *>(gmax);
    __shared__ long long s_next;
    __shared__ int s_hash;
    __shared__ uint32_t s_live[G];

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t *cbuf = cbuf_all + warp * BV_RD;
    const uint32_t lt_mask = (1u << lane) - 1u;
    uint32_t sat = 0;                                  // lane 0: rows capped in this item, flushed per item
    const int quads = p.D >> 2;                        // D % 4 == 0 (launcher)
    const BvTranspose tr(lane);
    const uint32_t planes_s = (uint32_t)__cvta_generic_to_shared(planes);
    if (threadIdx.x == 0) s_next = (long long)atomicAdd(p.item_ctr, 1ull);     // the first item

    for (;;) {
        // items are claimed one ahead, during the previous item's hashes (warp 0),
        // so no thread waits here on a global atomic
        if (p.n_sat && lane == 0 && sat) {             // the previous item's capped rows
            atomicAdd(p.n_sat, (unsigned long long)sat);
            sat = 0;
        }
        __syncthreads();                               // previous hashes done: planes free, s_next visible
        const long long item = s_next;
        if (threadIdx.x == 0) s_hash = 0;
        if (threadIdx.x < G) s_live[threadIdx.x] = 0;
        __syncthreads();                               // everyone has read s_next before warp 0 replaces it
        if (item >= p.n_items) break;
        const int64_t tile = item / p.n_hchunks;
        const int hc = (int)(item % p.n_hchunks);
        const int64_t row0 = tile * R;
        const int nr = (int)min((int64_t)R, p.n_rows - row0);
        const uint32_t j0 = (uint32_t)hc * p.hchunk, j1 = min(p.k, j0 + (uint32_t)p.hchunk);

        // ---- a5: stage the tile as bit planes + per-(column, group) maxima.
        //      Unit = (column quad, group, octet of 8 rows), octet fastest: 8
        //      words in, 4 columns x P plane bytes out; the 4 octet lanes of a
        //      (quad, group) combine their column maxima with two shuffles.
        //      BV_SB units per batch: all their loads are issued before any is
        //      used (one memory round trip per batch, not per unit)
        // unit = (column-quad pair, group, octet), octet fastest then columns: one
        // 8-byte load per row covers both quads, and a warp's load of a row index
        // touches 4 rows x 64 contiguous bytes; processed as two quads
        const int n_units = (quads / 2) * G * 4;
        // each thread ORs its live rows (nonzero in some column) per group in
        // registers; merged once per warp after staging
        uint32_t live_acc[G];
#pragma unroll
        for (int g = 0; g < G; g++) live_acc[g] = 0u;
        const int ncqp = quads / 2;                    // column-quad pairs per row
        // the delta-swap masks, kept in registers (LOP3 takes one immediate)
        uint32_t m1 = 0x55555555u, m1h = 0xAAAAAAAAu, m2 = 0x33333333u, m2h = 0xCCCCCCCCu, m4 = 0x0F0F0F0Fu, m4h = 0xF0F0F0F0u;
        asm volatile("" : "+r"(m1), "+r"(m1h), "+r"(m2), "+r"(m2h), "+r"(m4), "+r"(m4h));
        const uint8_t *xt = p.x + row0 * (int64_t)p.D;   // the tile's first row
        auto stage_load = [&](int u0, uint32_t (&wb)[BV_SB][2][8]) {
#pragma unroll
            for (int bi = 0; bi < BV_SB; bi++) {
                const int u = u0 + bi * NT;
                const int o = u & 3, cqp = (u >> 2) % ncqp, g = (u >> 2) / ncqp;
                const int rb = 32 * g + 8 * o;
                WMH_DASSERT(u >= n_units || (8 * cqp + 7 < p.D && g < G));
                // a tile holds < 2^32 bytes: 32-bit offsets from its first row
                const uint8_t *xr = xt + (uint32_t)(rb * p.D + 8 * cqp);
                if (u < n_units && rb + 8 <= nr) {     // the common case: the octet's rows all exist
#pragma unroll
                    for (int i = 0; i < 8; i++) {
                        const uint2 v = __ldg(reinterpret_cast<const uint2 *>(xr + (uint32_t)(i * p.D)));
                        wb[bi][0][i] = v.x;
                        wb[bi][1][i] = v.y;
                    }
                } else {
#pragma unroll
                    for (int i = 0; i < 8; i++) {
                        const bool ok = u < n_units && rb + i < nr;
                        WMH_DASSERT(!ok || row0 + rb + i < p.n_rows);
                        const uint2 v = ok ? __ldg(reinterpret_cast<const uint2 *>(xr + (uint32_t)(i * p.D))) : make_uint2(0u, 0u);
                        wb[bi][0][i] = v.x;
                        wb[bi][1][i] = v.y;
                    }
                }
            }
        };
        auto stage_proc = [&](int u0, uint32_t (&wb)[BV_SB][2][8]) {
#pragma unroll
            for (int bi = 0; bi < BV_SB; bi++) {
#pragma unroll
            for (int qq = 0; qq < 2; qq++) {
                const int u = u0 + bi * NT;
                if (u >= n_units) break;                 // uniform over the 4 octet lanes of a unit
                const int o = u & 3, g = (u >> 2) / ncqp, cq = 2 * ((u >> 2) % ncqp) + qq;
                uint32_t *w = wb[bi][qq];
                // 8x8 bit transposes of the 4 byte columns at once: delta swaps
                // across the 8 row words; afterwards w[b] = plane b (byte u4 =
                // column u4, bit i = row 8o + i)
                bv_swap<1>(w[0], w[1], m1, m1h); bv_swap<1>(w[2], w[3], m1, m1h);
                bv_swap<1>(w[4], w[5], m1, m1h); bv_swap<1>(w[6], w[7], m1, m1h);
                bv_swap<2>(w[0], w[2], m2, m2h); bv_swap<2>(w[1], w[3], m2, m2h);
                bv_swap<2>(w[4], w[6], m2, m2h); bv_swap<2>(w[5], w[7], m2, m2h);
#pragma unroll
                for (int i = 0; i < 4; i++)
                    if (i < P) bv_swap<4>(w[i], w[i + 4], m4, m4h);
                if (CLAMP) {                             // min(x, 2^P - 1): a set plane >= P sets planes 0..P-1
                    uint32_t hi = 0u;
#pragma unroll
                    for (int b = P; b < 8; b++) hi |= w[b];
#pragma unroll
                    for (int b = 0; b < P; b++) w[b] |= hi;
                }
                // 4x4 byte transpose across the 4 octet lanes: lane o then holds the
                // full 32-row plane words of column 4cq + o
                const unsigned am = __activemask();
                const uint32_t s1 = (o & 1) ? 0x3715u : 0x6240u, s2 = (o & 2) ? 0x3276u : 0x5410u;
                uint32_t pw[P];
#pragma unroll
                for (int b = 0; b < P; b++) {
                    uint32_t x = w[b];
                    x = bv_prmt(x, __shfl_xor_sync(am, x, 1), s1);
                    pw[b] = bv_prmt(x, __shfl_xor_sync(am, x, 2), s2);
                }
                const int c = 4 * cq + o;
                WMH_DASSERT(c < p.D && g < G);
                uint32_t *dst = planes + (size_t)c * W;
#pragma unroll
                for (int b = 0; b < P; b++) dst[BvLayout<P, G>::idx(g, b)] = pw[b];
                // the column's maximum over the group: bit descent on the planes
                uint32_t cand = 0u, mx = 0u;
#pragma unroll
                for (int b = 0; b < P; b++) cand |= pw[b];
#pragma unroll
                for (int gg = 0; gg < G; gg++) live_acc[gg] |= g == gg ? cand : 0u;   // rows of the group nonzero in this column
#pragma unroll
                for (int b = P - 1; b >= 0; b--) {
                    const uint32_t t = pw[b] & cand;
                    if (t) { cand = t; mx |= 1u << b; }
                }
                // clamped planes saturate at TOP: then only "some row >= TOP" is known,
                // so the flagged draws of this column keep testing (bv_slow is exact)
                gbytes[(size_t)c * sizeof(gm_t) + g] = (uint8_t)((CLAMP && mx == TOP) ? 0xFFu : mx);
            }
            }
        };
        // two batches of BV_SB units in flight: the next batch's loads are issued
        // before the current one is transposed
        {
            uint32_t bufA[BV_SB][2][8], bufB[BV_SB][2][8];
            int u0 = threadIdx.x;
            stage_load(u0, bufA);
            for (; u0 < n_units; u0 += 2 * BV_SB * NT) {
                const int u1 = u0 + BV_SB * NT;
                if (u1 < n_units) stage_load(u1, bufB);
                stage_proc(u0, bufA);
                if (u1 >= n_units) break;
                if (u1 + BV_SB * NT < n_units) stage_load(u1 + BV_SB * NT, bufA);
                stage_proc(u1, bufB);
            }
        }
        {
#pragma unroll
            for (int gg = 0; gg < G; gg++) {
                const uint32_t lv = __reduce_or_sync(0xFFFFFFFFu, live_acc[gg]);
                if (lane == 0 && lv) atomicOr(&s_live[gg], lv);
            }
        }
        __syncthreads();

        // ---- warp 0 claims the next item now and warms L2 with its rows
        if (warp == 0) {
            long long nx = 0;
            if (lane == 0) nx = (long long)atomicAdd(p.item_ctr, 1ull);
            nx = __shfl_sync(0xFFFFFFFFu, nx, 0);
            if (lane == 0) s_next = nx;
            if (nx < p.n_items) {
                const int64_t nrow0 = (nx / p.n_hchunks) * R;
                const int64_t nbytes = min((int64_t)R, p.n_rows - nrow0) * (int64_t)p.D;
                const char *base = reinterpret_cast<const char *>(p.x + nrow0 * (int64_t)p.D);
                if (p.bulk_pf) {
                    // the tile's rows are contiguous: one TMA bulk prefetch per lane
                    // (cp.async.bulk.prefetch.L2, 16-byte granules of its share)
                    const int64_t per = ((nbytes + 31) / 32 + 15) & ~(int64_t)15;
                    const int64_t off = (int64_t)lane * per;
                    const int64_t sz = min(per, nbytes - off) & ~(int64_t)15;
                    if (sz > 0)
                        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(base + off), "r"((uint32_t)sz) : "memory");
                } else {
                    for (int64_t off = (int64_t)lane * 128; off < nbytes; off += 32 * 128)
                        asm volatile("prefetch.global.L2 [%0];" ::"l"(base + off));
                }
            }
        }

        // ---- hashes: a warp claims blocks of BV_HB consecutive hashes (the next
        //      block one block ahead).  Lane = row: the block's results of rows
        //      32g + lane are kept packed in registers (acc[g], 2 per word, shifted
        //      in hash by hash) and flushed with one 16-byte store per row
        //      The item's last ~4 hashes per warp are claimed in blocks of 4 (the
        //      barrier tail behind the slowest warp is one block long).
        const uint32_t span = j1 - j0, n_tail = 4u * (NT / 32);
        const uint32_t tail0 = j0 + (span > n_tail ? (span - n_tail) & ~(uint32_t)(BV_HB - 1) : 0u);
        const uint32_t nb_full = (tail0 - j0) / BV_HB;
        auto grab = [&]() {
            int bb = 0;
            if (lane == 0) bb = atomicAdd(&s_hash, 1);
            const uint32_t b = (uint32_t)__shfl_sync(0xFFFFFFFFu, bb, 0);
            return min(j1, b < nb_full ? j0 + (uint32_t)BV_HB * b : tail0 + 4u * (b - nb_full));
        };
        auto block_end = [&](uint32_t jb_) { return min(j1, jb_ + (jb_ < tail0 ? (uint32_t)BV_HB : 4u)); };
        uint32_t pend0[G], dead[G];
#pragma unroll
        for (int g = 0; g < G; g++) {
            const uint32_t valid = 32 * g + 32 <= nr ? 0xFFFFFFFFu : (32 * g >= nr ? 0u : (1u << (nr - 32 * g)) - 1u);
            pend0[g] = s_live[g] & valid;
            dead[g] = valid & ~s_live[g];
        }
        uint32_t n_dead = 0;                           // all-zero rows: h = cap at once (R12)
#pragma unroll
        for (int g = 0; g < G; g++) n_dead += __popc(dead[g]);
        uint32_t acc[G][BV_HB / 2];
#pragma unroll
        for (int g = 0; g < G; g++)
#pragma unroll
            for (int i = 0; i < BV_HB / 2; i++) acc[g][i] = 0u;
        uint32_t jb = grab();                          // current block [jb, je)
        uint32_t je = block_end(jb);
        uint32_t jb_next = jb < j1 ? grab() : j1;
        uint32_t j = jb;
        // draw words: lane holds t = tb + 32 s + lane (s < BV_DPL) of the current
        // round, of the next round, and of the next hash's first round
        uint32_t nw[BV_DPL];
#pragma unroll
        for (int s = 0; s < BV_DPL; s++) nw[s] = 0u;
        if (j < j1) {
            WMH_DASSERT(j < p.k);
            const uint32_t *t0 = p.table + (int64_t)j * BV_T0;
#pragma unroll
            for (int s = 0; s < BV_DPL; s++) nw[s] = __ldg(t0 + 32 * s + lane);
        }
        while (j < j1) {
            const uint32_t jn = j + 1 < je ? j + 1 : jb_next;
            const uint32_t tj = j * (uint32_t)BV_T0;       // this hash's table row (k * BV_T0 < 2^32)
            uint32_t cw[BV_DPL];                       // this round's draw words
#pragma unroll
            for (int s = 0; s < BV_DPL; s++) cw[s] = nw[s];
            if (jn < j1) {                             // one hash ahead: its first round
                const uint32_t tn = jn * (uint32_t)BV_T0;
#pragma unroll
                for (int s = 0; s < BV_DPL; s++) nw[s] = __ldg(p.table + (tn + 32 * s + lane));
            }
            // h of row 32g + lane; rows without a green draw before the cap (and
            // all-zero rows) keep h = cap
            uint32_t hcur[G];
            uint32_t pend[G];
#pragma unroll
            for (int g = 0; g < G; g++) {
                hcur[g] = p.cap;
                pend[g] = pend0[g];
            }
            sat += (lane == 0) ? n_dead : 0u;
            for (uint32_t tb = 0;; tb += BV_RD) {
                uint32_t anyp = 0;
#pragma unroll
                for (int g = 0; g < G; g++) anyp |= pend[g];
                if (!anyp) break;
                uint32_t w[BV_DPL];
#pragma unroll
                for (int s = 0; s < BV_DPL; s++) w[s] = cw[s];
                if (tb >= (uint32_t)BV_T0) {           // beyond the table (rare): draw them here
                    const uint64_t keyj = p.S ^ ((uint64_t)j << 32);
#pragma unroll
                    for (int s = 0; s < BV_DPL; s++) {
                        const uint32_t t = tb + 32 * s + lane;
                        w[s] = bv_word(mulhi_range(splitmix64(keyj ^ (uint64_t)t), p.M), p.pack, p.uni_m, t, p.cap);
                    }
                }
                if (tb + BV_RD < (uint32_t)BV_T0) {    // prefetch the next round
#pragma unroll
                    for (int s = 0; s < BV_DPL; s++) cw[s] = __ldg(p.table + (tj + tb + BV_RD + 32 * s + lane));
                }
                // ---- a5/a6 screen: a draw is needed when its offset is below the
                //      column maximum of a pending group; the needed draws of the
                //      round are compacted in draw order into the warp's list
                //      (entry = word << 7 | t - tb)
                uint32_t gms[BV_DPL];                  // all column maxima loaded before any list store
#pragma unroll
                for (int s = 0; s < BV_DPL; s++) {
                    WMH_DASSERT((w[s] >> 8) < (uint32_t)p.D);
                    gms[s] = (uint32_t)gmax[w[s] >> 8];
                }
                uint32_t total = 0;
#pragma unroll
                for (int s = 0; s < BV_DPL; s++) {
                    const uint32_t off = w[s] & 0xFFu, gm = gms[s];
                    bool need = false;
#pragma unroll
                    for (int g = 0; g < G; g++) need |= pend[g] != 0u && off < ((gm >> (8 * g)) & 0xFFu);
                    const uint32_t bal = __ballot_sync(0xFFFFFFFFu, need);
                    if (need) cbuf[total + __popc(bal & lt_mask)] = (w[s] << 7) | (uint32_t)(32 * s + lane);
                    total += __popc(bal);
                }
                if (total == 0u) {                     // draws at t >= cap are never needed (word 0xFF)
                    if (tb + BV_RD >= p.cap) {         // a8: no green draw before the cap
#pragma unroll
                        for (int g = 0; g < G; g++) sat += (lane == 0) ? __popc(pend[g]) : 0;
                        break;
                    }
                    continue;
                }
                __syncwarp();
                // ---- test the needed draws, 32 at a time (lane = draw), in draw order
                for (uint32_t base = 0; base < total; base += 32) {
                    const bool valid = base + lane < total;
                    const uint32_t e = valid ? cbuf[base + lane] : 0u;
                    const uint32_t we = e >> 7, toff = e & 127u;
                    uint32_t mk[G];
                    const bool slow = bv_test_c<P, G, CLAMP>(planes_s, we, valid, mk);
                    if (CLAMP && slow) {               // rare, divergent
#pragma unroll
                        for (int g = 0; g < G; g++) mk[g] = bv_test_slow<P, G>(p, planes_s, gmax, row0, we, pend[g], g);
                    }
                    // ---- a8: the first green draw of each pending row: one transpose
                    //      per group gives lane = row the first list position i
                    //      with a green; its draw is tb + toff_i
                    uint32_t u[G], anyu = 0u;
#pragma unroll
                    for (int g = 0; g < G; g++) {
                        u[g] = mk[g] & pend[g];
                        anyu |= u[g];
                    }
                    if (__any_sync(0xFFFFFFFFu, anyu != 0u)) {
                        uint32_t wt[G];
#pragma unroll
                        for (int g = 0; g < G; g++) wt[g] = tr(u[g]);   // bit i: list entry base + i green for row lane
#pragma unroll
                        for (int g = 0; g < G; g++) {
                            const int i = __ffs(wt[g]) - 1;
                            const uint32_t ti = __shfl_sync(0xFFFFFFFFu, toff, i & 31);
                            if (wt[g]) hcur[g] = tb + ti + 1u;
                            pend[g] &= ~__ballot_sync(0xFFFFFFFFu, wt[g] != 0u);
                        }
                    }
                }
                __syncwarp();                          // the list is rewritten next round
            }
            // shift the hash's results in: slot BV_HB - 1 is the newest
#pragma unroll
            for (int g = 0; g < G; g++) {
#pragma unroll
                for (int i = 0; i < BV_HB / 2 - 1; i++) acc[g][i] = bv_prmt(acc[g][i], acc[g][i + 1], 0x5432u);
                acc[g][BV_HB / 2 - 1] = bv_prmt(acc[g][BV_HB / 2 - 1], hcur[g], 0x5432u);
            }
            if (j + 1 == je) {
                // ---- a9: flush the block: row r's hashes jb..je-1 are contiguous in sig
                const int nh = (int)(je - jb);
                WMH_DASSERT(nh >= 1 && nh <= BV_HB);
                for (int u = nh; u < BV_HB; u++) {     // a short block: align hash jb to slot 0
#pragma unroll
                    for (int g = 0; g < G; g++) {
#pragma unroll
                        for (int i = 0; i < BV_HB / 2 - 1; i++) acc[g][i] = bv_prmt(acc[g][i], acc[g][i + 1], 0x5432u);
                        acc[g][BV_HB / 2 - 1] = bv_prmt(acc[g][BV_HB / 2 - 1], 0u, 0x5432u);
                    }
                }
#pragma unroll
                for (int g = 0; g < G; g++) {
                    const int r = 32 * g + lane;
                    if (r >= nr) continue;
                    const int64_t e = (row0 + r) * (int64_t)p.k + jb;
                    WMH_DASSERT(e + nh <= p.n_rows * (int64_t)p.k);
                    if (nh == BV_HB && p.vec_flush) {
                        static_assert(BV_HB == 8, "the vector flush packs 8 hashes");
                        if (p.sigb == 2) {
                            uint16_t *ptr = reinterpret_cast<uint16_t *>(p.sig) + e;
                            if (p.vec_flush == 2) {
                                *reinterpret_cast<uint4 *>(ptr) = make_uint4(acc[g][0], acc[g][1], acc[g][2], acc[g][3]);
                            } else {
                                reinterpret_cast<uint2 *>(ptr)[0] = make_uint2(acc[g][0], acc[g][1]);
                                reinterpret_cast<uint2 *>(ptr)[1] = make_uint2(acc[g][2], acc[g][3]);
                            }
                        } else {
                            uint8_t *ptr = reinterpret_cast<uint8_t *>(p.sig) + e;
                            *reinterpret_cast<uint2 *>(ptr) = make_uint2(bv_prmt(acc[g][0], acc[g][1], 0x6420u),
                                                                         bv_prmt(acc[g][2], acc[g][3], 0x6420u));
                        }
                    } else if (nh == 4 && p.vec_flush) {   // a tail block (jb - j0 = 0 mod 4)
                        if (p.sigb == 2) *reinterpret_cast<uint2 *>(reinterpret_cast<uint16_t *>(p.sig) + e) = make_uint2(acc[g][0], acc[g][1]);
                        else *reinterpret_cast<uint32_t *>(reinterpret_cast<uint8_t *>(p.sig) + e) = bv_prmt(acc[g][0], acc[g][1], 0x6420u);
                    } else {
#pragma unroll
                        for (int u = 0; u < BV_HB; u++) {
                            if (u >= nh) break;
                            const uint32_t v = (acc[g][u >> 1] >> (16 * (u & 1))) & 0xFFFFu;
                            if (p.sigb == 2) reinterpret_cast<uint16_t *>(p.sig)[e + u] = (uint16_t)v;
                            else reinterpret_cast<uint8_t *>(p.sig)[e + u] = (uint8_t)v;
                        }
                    }
                }
                __syncwarp();
                jb = jb_next;
                je = block_end(jb);
                jb_next = jb < j1 ? grab() : j1;
            }
            j = jn;
        }
    }
    if (p.n_sat && lane == 0 && sat) atomicAdd(p.n_sat, (unsigned long long)sat);
}

static size_t bv_smem(int D, int G, int P, int NT) {
    const size_t gm_bytes = (size_t)D * (G == 1 ? 1 : G == 2 ? 2 : 4);
    return (size_t)D * G * P * 4 + ((gm_bytes + 15) & ~(size_t)15) + (size_t)(NT / 32) * BV_RD * 4;
}

template <int P, int G, bool CLAMP, int NT>
static void bv_launch(const BvParams &p, size_t smem, int grid, cudaStream_t s) {
    auto kern = hash_bitslice_kernel<P, G, CLAMP, NT>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kernel_timer_begin(s);
    kern<<<grid, NT, smem, s>>>(p);
    kernel_timer_end(s);
}

template <int P, bool CLAMP>
static void bv_launch_g(int G, int NT, const BvParams &p, size_t smem, int grid, cudaStream_t s) {
    (void)NT;                                    // BV_NT threads
    if (G == 4) bv_launch<P, 4, CLAMP, BV_NT>(p, smem, grid, s);
    else if (G == 2) bv_launch<P, 2, CLAMP, BV_NT>(p, smem, grid, s);
    else bv_launch<P, 1, CLAMP, BV_NT>(p, smem, grid, s);
}

template <int P>
static void bv_launch_p(int G, bool clamp, int NT, const BvParams &p, size_t smem, int grid, cudaStream_t s) {
    if (clamp) {
        if constexpr (P >= 4 && P < 8) bv_launch_g<P, true>(G, NT, p, smem, grid, s);
        return;
    }
    bv_launch_g<P, false>(G, NT, p, smem, grid, s);
}

#define WMH_BV_P_SWITCH(PV, CALL) \
    switch (PV) {                 \
        case 1: CALL(1); break;   \
        case 2: CALL(2); break;   \
        case 3: CALL(3); break;   \
        case 4: CALL(4); break;   \
        case 5: CALL(5); break;   \
        case 6: CALL(6); break;   \
        case 7: CALL(7); break;   \
        default: CALL(8); break;  \
    }

// Shape of the tile for a layout: planes P (clamped: NB - 1), groups G of 32
// rows, threads per CTA NT and CTAs per SM (512 -> 1, 256 -> 2); G = 0 when
// the rows are too long for even one group of exact planes.
struct BvShape {
    int P, G;
    bool clamp;
    int NT, ctas;
};

static BvShape bv_shape(const HashArgs &a) {
    const int D = (int)a.rows.dim;
    const int NB = 32 - __builtin_clz(a.L->max_bound);
    int dev = 0;
    cudaGetDevice(&dev);
    int smem_optin = 0;
    cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    static const int g_env = getenv("WMH_BV_GROUPS") ? atoi(getenv("WMH_BV_GROUPS")) : 0;
    const int gmax_try = (g_env == 1 || g_env == 2 || g_env == 4) ? g_env : 4;
    // one BV_NT-thread CTA per SM: the planes fill shared memory (measured: two
    // 256-thread CTAs with one group each 15.5 vs 14.1 ms)
    const int ctas = 1, NT = BV_NT;
    const size_t budget = (size_t)smem_optin - 64;
    // WMH_BV_PLANES=P (4 <= P < NB): clamp to P planes whenever they fit two groups
    static const int p_env = getenv("WMH_BV_PLANES") ? atoi(getenv("WMH_BV_PLANES")) : 0;
    if (p_env >= 4 && p_env < NB && p_env < 8) {
        for (int G = gmax_try; G >= 1; G /= 2)
            if (bv_smem(D, G, p_env, NT) <= budget) return {p_env, G, true, NT, ctas};
    }
    // A thin tail of large weights: clamp to the fewest planes P >= 4 for which a
    // 32-row group holds a weight >= 2^P - 1 with probability <= 1% (prepare's
    // sampled fraction f: 1 - (1 - f)^32); the draws in the top cells of those
    // groups' columns are tested on the rows' bytes.  Shorter chains, smaller
    // tiles (c5: P = 5 of NB = 7, 39.6 vs 42.0 ms on 4M rows; P = 4 has f = 0.3%
    // and measured 70.7 ms).
    if (a.L->value_cells > 0 && NB > 4) {
        for (int q = 4; q < NB && q < 8; q++) {
            const double f = (double)a.L->value_ge[q] / (double)a.L->value_cells;
            if (1.0 - pow(1.0 - f, 32.0) > 0.01) continue;
            for (int G = gmax_try; G >= 1; G /= 2)
                if (bv_smem(D, G, q, NT) <= budget) return {q, G, true, NT, ctas};
            break;
        }
    }
    for (int G = gmax_try; G >= 1; G /= 2) {
        if (bv_smem(D, G, NB, NT) <= budget) return {NB, G, false, NT, ctas};
        // one plane fewer (clamped) when it buys this group count
        if (G >= 2 && NB >= 5 && bv_smem(D, G, NB - 1, NT) <= budget) return {NB - 1, G, true, NT, ctas};
    }
    return {NB, 0, false, NT, ctas};
}

bool bitslice_handles(const HashArgs &a) {
    const int D = (int)a.rows.dim;
    if (a.rows.kind != WMH_DENSE || (D & 7) || ((uintptr_t)a.rows.dense & 7)) return false;
    if ((a.L->flags & WMH_LAYOUT_WIDE) || weight_bytes(a.rows) != 1 || a.L->max_bound == 0 || a.L->max_bound > 255) return false;
    if ((uint64_t)D >= (1ull << 16)) return false;     // list entries: (c << 8 | off) << 7 | t - tb in 31 bits
    return bv_shape(a).G >= 1;
}

wmh_status launch_hash_bitslice(const HashArgs &a, bool *handled) {
    *handled = false;
    if (!bitslice_handles(a)) return WMH_OK;
    const int D = (int)a.rows.dim;
    const BvShape sh = bv_shape(a);
    const int G = sh.G, P = sh.P, R = 32 * G;
    const size_t smem = bv_smem(D, G, P, sh.NT);
    *handled = true;

    const int64_t n_tiles = (a.rows.n_rows + R - 1) / R;
    const int sms = num_sms();
    // >= 8 items per SM for balance, but >= WMH_MIN_HCHUNK hashes per item: each
    // item stages its whole tile, so small batches must not slice k too thin
    static const int min_hc = getenv("WMH_MIN_HCHUNK") ? std::max(8, atoi(getenv("WMH_MIN_HCHUNK"))) : 128;
    int n_hchunks = (int)std::max((int64_t)1, std::min((int64_t)(a.k + min_hc - 1) / min_hc, ((int64_t)sms * sh.ctas * 8 + n_tiles - 1) / n_tiles));
    const int hchunk = (int)(((a.k + n_hchunks - 1) / n_hchunks + BV_HB - 1) / BV_HB * BV_HB);
    n_hchunks = (int)((a.k + hchunk - 1) / hchunk);

    uint8_t *scratch = nullptr;
    const size_t tab_bytes = (size_t)a.k * BV_T0 * sizeof(uint32_t);
    WMH_CUDA_TRY(cudaMallocAsync((void **)&scratch, tab_bytes + 256, a.stream), "bitslice scratch alloc");
    uint32_t *table = reinterpret_cast<uint32_t *>(scratch);
    unsigned long long *ctr = reinterpret_cast<unsigned long long *>(scratch + tab_bytes);
    WMH_CUDA_TRY(cudaMemsetAsync(ctr, 0, sizeof(unsigned long long), a.stream), "bitslice counter memset");
    const uint32_t uni_m = (a.L->flags & WMH_LAYOUT_UNIFORM) ? a.L->uniform_m : 0u;
    {
        const int64_t total = (int64_t)a.k * BV_T0;
        const int blocks = (int)std::min((int64_t)sms * 8, (total + 255) / 256);
        bv_table_kernel<<<blocks, 256, 0, a.stream>>>(table, a.k, a.S, (uint32_t)a.L->M, a.L->cell_pack, uni_m, a.cap,
                                                      a.isgreen_bsearch ? a.L->comp_to_m : nullptr, (uint32_t)D);
        count_launch();
        const cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) { cudaFreeAsync(scratch, a.stream); return cuda_fail(e, "bitslice table launch"); }
    }

    BvParams p;
    p.x = a.rows.dense;
    p.n_rows = a.rows.n_rows;
    p.D = D;
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
    // WMH_BV_NO_BULKPF: the per-line prefetch loop instead (A/B)
    p.bulk_pf = ((uintptr_t)a.rows.dense & 15) == 0 && (D & 15) == 0 && !getenv("WMH_BV_NO_BULKPF");
    const int grid = (int)std::min((int64_t)sms * sh.ctas, p.n_items);
#define WMH_BV_GO(V) bv_launch_p<V>(G, sh.clamp, sh.NT, p, smem, grid, a.stream)
    WMH_BV_P_SWITCH(P, WMH_BV_GO)
#undef WMH_BV_GO
    WMH_LAUNCH_CHECK("hash_bitslice launch");
    if (getenv("WMH_TILED_STATS"))
        fprintf(stderr, "[wmh bitslice] P=%d clamp=%d G=%d NT=%d grid=%d items=%lld hchunk=%d smem=%zu\n", P, (int)sh.clamp, G,
                sh.NT, grid, (long long)p.n_items, hchunk, smem);
    cudaFreeAsync(scratch, a.stream);
    return WMH_OK;
}

}  // namespace wmh
