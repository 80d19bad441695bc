// hash_tiled_cm.cu -- WMH_ALGO_TILED for dense rows, column-major tile (default).
//
// Same algorithm as hash_tiled.cu (each draw r_t of hash j is shared by the
// tile's rows, because the draw stream does not depend on x), but
// the tile is stored column-major -- x[row][c] at byte c * Rp + row -- so
// one 32-bit shared load returns column c of FOUR rows.  That makes the first
// round of every hash (draws t = 0..31, which every row must see and which
// resolve ~80% of the rows at s ~ 0.05) a SIMD-within-a-register test:
//
//   green(x, off)  <=>  x > off  <=>  x + (255 - off) >= 256
//
// computed for 4 bytes at once as the carry out of bit 7:
//   s = (a & 0x7F7F7F7F) + K,  K = ((255 - off) & 0x7F) * 0x01010101
//   g = MAJ(a, B, s)           B = (255 - off) * 0x01010101    (one LOP3)
//   m = PRMT(g, msb-replicate)  -> 0xFF in every green byte
//   h = (h & ~m) | (i * 0x01010101 & m)   (draws visited in descending i)
// -- one LDS and ~8 instructions per draw for 4 rows.  The tile holds
// R = 32 * 4 / P rows (P = 1, 2, 4) so that round 0 is exactly one (4-row word,
// 32/P-draw part) unit per lane.  Rows still without a green continue on the
// warp's pending list (lane = row, C draws per re-queue, then draw-parallel
// stragglers) with addresses c * Rp + row.  Results go to a per-warp shared
// row h[R] and are flushed to the signatures once per hash.  First green t
// gives h = t + 1 (Alg. 3 / Def.); no green before the cap gives
// h = cap (reading R9); all-zero rows get cap (R12).
#include <stdio.h>
#include <stdlib.h>

#include <type_traits>

#include "common.cuh"

namespace wmh {

constexpr int CM_NT = 512;
constexpr int CM_NW = CM_NT / 32;
constexpr int CM_STRAG = 4;
constexpr int CM_HB = 8;                 // hashes per claimed block (results flushed 8 per row)

struct CmParams {
    const uint8_t *x;
    int64_t n_rows;
    int D, R, Rp;                // dim, rows per tile (128/64/32), column stride (bytes, Rp/4 odd)
    int n_hchunks, hchunk;
    int64_t n_items;
    uint32_t k, cap, M, uni_m;
    uint64_t S;
    int chunk;                   // 0 = auto (from the tile's effective sparsity)
    int vec_flush;               // k % 4 == 0 and sig aligned: 4-hash row stores
    const uint32_t *table;       // [k][T0] packed draws (c * Rp) << 8 | nb, nb = 255 - off (0 at t >= cap)
    const uint32_t *pack;
    void *sig;
    unsigned long long *n_sat;
    unsigned long long *item_ctr;
};

// A draw packed for the tile: (c * Rp) << 8 | nb with nb = 255 - (r - CompToM[c]),
// and nb = 0 (never green: x + nb < 256) for t >= cap.  green(x) <=> x + nb >= 256
// <=> x > nb ^ 0xFF.
__device__ __forceinline__ uint32_t cm_pack(uint32_t r, const uint32_t *pack, uint32_t uni_m, uint32_t Rp, uint32_t t,
                                            uint32_t cap) {
    const uint2 d = unpack_cell(cell_of(r, pack, uni_m));
    return ((d.x * Rp) << 8) | (t < cap ? 255u - d.y : 0u);
}

__device__ __forceinline__ uint32_t cm_late(const CmParams &p, uint64_t keyj, uint32_t t) {
    return cm_pack(mulhi_range(splitmix64(keyj ^ (uint64_t)t), p.M), p.pack, p.uni_m, (uint32_t)p.Rp, t, p.cap);
}

// TW = 1: one packed word per draw; TW = 2: (c * Rp, nb in every byte) -- the
// SWAR constant B ready, two fewer ALU ops per draw-word test for twice the
// shared-load bytes (the 128-row tile is ALU-bound, the 32-row tile load-bound)
template <int TW>
__device__ __forceinline__ void cm_put(uint32_t *dst, uint32_t pw) {
    if (TW == 1) dst[0] = pw;
    else *reinterpret_cast<uint2 *>(dst) = make_uint2(pw >> 8, (pw & 0xFFu) * 0x01010101u);
}

template <int TW>
__global__ void cm_table_kernel(uint32_t *__restrict__ table, uint32_t k, uint64_t S, uint32_t M,
                                const uint32_t *__restrict__ pack, uint32_t uni_m, uint32_t Rp, uint32_t cap) {
    const int64_t total = (int64_t)k * T0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t j = (uint32_t)(i / T0), t = (uint32_t)(i % T0);
        cm_put<TW>(table + i * TW, cm_pack(draw_r(S, j, t, M), pack, uni_m, Rp, t, cap));
    }
}

// column offset and off of draw t from a TW-word table
template <int TW>
__device__ __forceinline__ uint2 cm_get(const uint32_t *buf, uint32_t t) {
    if (TW == 1) {
        const uint32_t pw = buf[t];
        return make_uint2(pw >> 8, (pw & 0xFFu) ^ 0xFFu);
    }
    const uint2 d = *reinterpret_cast<const uint2 *>(buf + 2 * t);
    return make_uint2(d.x, (d.y & 0xFFu) ^ 0xFFu);
}

__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
    uint32_t d;
    asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(sel));
    return d;
}

// Rounds 1.. over the pending list: lane = row, C draws per re-queue;
// results to the warp's shared row hres[].
template <int C, int TW>
__device__ __forceinline__ int cm_rounds(const CmParams &p, const uint32_t *buf, uint32_t *win, const uint8_t *xs,
                                         uint64_t keyj, uint16_t *hres, const uint16_t *&cur, uint16_t *own0,
                                         uint16_t *own1, int npend, uint32_t *q_io) {
    const int lane = threadIdx.x & 31;
    uint32_t q = *q_io;
    int flip = 0;
    while (npend > CM_STRAG && q * 32 < p.cap) {
        const uint32_t *src;
        if (q * 32 < (uint32_t)T0) {
            src = buf + q * 32 * TW;
        } else {
            const uint32_t d = cm_late(p, keyj, q * 32 + lane);
            __syncwarp();
            cm_put<TW>(win + lane * TW, d);
            __syncwarp();
            src = win;
        }
#pragma unroll
        for (int sub = 0; sub < 32 / C; sub++) {
            if (npend == 0) break;
            uint32_t dc[C], doff[C];
#pragma unroll
            for (int i = 0; i < C * TW / 4; i++) {     // 16-byte loads: four (TW = 1) or two draws
                const uint4 v = reinterpret_cast<const uint4 *>(src + sub * C * TW)[i];
                const uint32_t w4[4] = {v.x, v.y, v.z, v.w};
                if (TW == 1) {
#pragma unroll
                    for (int u = 0; u < 4; u++) {
                        dc[4 * i + u] = w4[u] >> 8;
                        doff[4 * i + u] = (w4[u] & 0xFFu) ^ 0xFFu;   // off (255 at t >= cap: never green)
                    }
                } else {
#pragma unroll
                    for (int u = 0; u < 2; u++) {
                        dc[2 * i + u] = w4[2 * u];
                        doff[2 * i + u] = (w4[2 * u + 1] & 0xFFu) ^ 0xFFu;
                    }
                }
            }
            uint16_t *nxt = flip ? own1 : own0;
            flip ^= 1;
            int nn = 0;
            for (int base = 0; base < npend; base += 32) {
                const int i = base + lane;
                const bool active = i < npend;
                const int r = active ? cur[i] : 0;
                uint32_t h = C;
                if (active) {
                    constexpr int NCH = C >= 16 ? 4 : 2;
                    uint32_t hc[NCH];
#pragma unroll
                    for (int c = 0; c < NCH; c++) hc[c] = C;
#pragma unroll
                    for (int tt = C - 1; tt >= 0; tt--) {
                        const uint32_t v = xs[dc[tt] + r];
                        hc[tt % NCH] = (v > doff[tt]) ? (uint32_t)tt : hc[tt % NCH];
                    }
                    h = hc[0];
#pragma unroll
                    for (int c = 1; c < NCH; c++) h = min(h, hc[c]);
                }
                const bool still = active && h == C;
                if (active && !still) hres[r] = (uint16_t)(q * 32 + sub * C + h + 1);
                const unsigned m = __ballot_sync(0xFFFFFFFFu, still);
                if (still) nxt[nn + __popc(m & ((1u << lane) - 1))] = (uint16_t)r;
                nn += __popc(m);
            }
            __syncwarp();
            cur = nxt;
            npend = nn;
        }
        q++;
    }
    *q_io = q;
    return npend;
}

template <int SIGB, int P, int NR0, int TW>
__global__ void __launch_bounds__(CM_NT, 1) hash_tiled_cm_kernel(const CmParams p) {
    // rows, 4-row words (NWD * P == 32), draws per part of the NR0 SWAR rounds
    constexpr int R = 128 / P, NWD = R / 4, PD = 32 * NR0 / P;
    extern __shared__ __align__(16) uint32_t smem[];
    const int Rp = p.Rp;
    uint8_t *xs = reinterpret_cast<uint8_t *>(smem);                               // [D][Rp]
    const size_t xs_bytes = ((size_t)p.D * Rp + 15) & ~(size_t)15;
    uint32_t *sbuf_all = reinterpret_cast<uint32_t *>(xs + xs_bytes);               // [NW][T0][TW] draws
    uint32_t *swin_all = sbuf_all + CM_NW * T0 * TW;                                // [NW][32][TW]
    uint32_t *spart_all = swin_all + CM_NW * 32 * TW;                               // [NW][32] partial h4
    uint16_t *hres_all = reinterpret_cast<uint16_t *>(spart_all + CM_NW * 32);      // [NW][HB][R] results
    uint16_t *spend_all = hres_all + CM_NW * CM_HB * R;                             // [NW][2][R]
    uint8_t *sflag4 = reinterpret_cast<uint8_t *>(spend_all + CM_NW * 2 * R);       // [NWD] live-row nibbles
    __shared__ long long s_item, s_next;
    __shared__ int s_hash, s_nalive;
    __shared__ unsigned long long s_xsum;

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t *sbuf = sbuf_all + warp * T0 * TW;
    uint32_t *swin = swin_all + warp * 32 * TW;
    uint32_t *spart = spart_all + warp * 32;
    uint16_t *hres_blk = hres_all + warp * CM_HB * R;                              // [HB][R]
    uint16_t *own0 = spend_all + warp * 2 * R, *own1 = own0 + R;
    unsigned long long sat = 0;
    const int words = p.D >> 2;                        // D % 4 == 0 (launcher)
    if (threadIdx.x == 0) s_next = (long long)atomicAdd(p.item_ctr, 1ull);

    for (;;) {
        __syncthreads();
        if (threadIdx.x == 0) {
            s_item = s_next;
            s_next = (long long)atomicAdd(p.item_ctr, 1ull);
            s_hash = 0;
            s_xsum = 0;
            s_nalive = 0;
        }
        __syncthreads();
        const long long item = s_item;
        if (item >= p.n_items) break;
        if (s_next < p.n_items) {                      // warm L2 with the next item's rows
            const int64_t nrow0 = (s_next / p.n_hchunks) * R;
            const int64_t nbytes = min((int64_t)R, p.n_rows - nrow0) * (int64_t)p.D;
            const char *base = reinterpret_cast<const char *>(p.x + nrow0 * (int64_t)p.D);
            for (int64_t off = (int64_t)threadIdx.x * 128; off < nbytes; off += (int64_t)CM_NT * 128)
                asm volatile("prefetch.global.L2 [%0];" ::"l"(base + off));
        }
        const int64_t tile = item / p.n_hchunks;
        const int hc = (int)(item % p.n_hchunks);
        const int64_t row0 = tile * R;
        const int nr = (int)min((int64_t)R, p.n_rows - row0);
        const uint32_t j0 = (uint32_t)hc * p.hchunk, j1 = min(p.k, j0 + (uint32_t)p.hchunk);

        // ---- a5: stage transposed: 4 rows x 4 columns per lane, 8 PRMTs --------
        unsigned long long wsum = 0;                   // this warp's row sums / live rows: one
        int walive = 0;                                // shared atomic per warp, not per row
        for (int g = warp; g < NWD; g += CM_NW) {
            const uint32_t *rp[4];
            bool ok[4];
#pragma unroll
            for (int b = 0; b < 4; b++) {
                ok[b] = 4 * g + b < nr;
                rp[b] = reinterpret_cast<const uint32_t *>(p.x + (row0 + (ok[b] ? 4 * g + b : 0)) * (int64_t)p.D);
            }
            uint32_t acc[4] = {0, 0, 0, 0};
            const int st = Rp >> 2;                    // words per column
#pragma unroll 2
            for (int cg = lane; cg < words; cg += 32) {
                uint32_t v[4];
#pragma unroll
                for (int b = 0; b < 4; b++) {
                    v[b] = ok[b] ? __ldg(rp[b] + cg) : 0u;
                    acc[b] = __dp4a(v[b], 0x01010101u, acc[b]);
                }
                const uint32_t t0 = prmt(v[0], v[1], 0x5140), t1 = prmt(v[0], v[1], 0x7362);
                const uint32_t t2 = prmt(v[2], v[3], 0x5140), t3 = prmt(v[2], v[3], 0x7362);
                uint32_t *col = reinterpret_cast<uint32_t *>(xs + (size_t)(4 * cg) * Rp) + g;
                col[0] = prmt(t0, t2, 0x5410);
                col[st] = prmt(t0, t2, 0x7632);
                col[2 * st] = prmt(t1, t3, 0x5410);
                col[3 * st] = prmt(t1, t3, 0x7632);
            }
            uint32_t live4 = 0;
#pragma unroll
            for (int b = 0; b < 4; b++) {
                uint32_t a = acc[b];
                for (int o = 16; o; o >>= 1) a += __shfl_xor_sync(0xFFFFFFFFu, a, o);
                if (a) live4 |= 1u << b;
                wsum += a;
                walive += a != 0;
            }
            if (lane == 0) sflag4[g] = (uint8_t)live4;
        }
        if (lane == 0 && walive) {
            atomicAdd(&s_xsum, wsum);
            atomicAdd(&s_nalive, walive);
        }
        __syncthreads();
        const int nalive = s_nalive;
        int C = p.chunk;
        if (C == 0) {
            const double s = nalive ? (double)s_xsum / ((double)nalive * (double)p.M) : 1.0;
            C = s > 0.2 ? 8 : s > 0.1 ? 16 : 32;
        }

        // ---- hashes: a warp claims blocks of CM_HB consecutive hashes (the next
        //      block one block ahead, hiding the shared atomic), prefetches the
        //      next hash's draws, and flushes a block's results with one store
        //      per row -------------------------------------------------------------
        auto grab = [&]() {
            int bb = 0;
            if (lane == 0) bb = atomicAdd(&s_hash, 1);
            return min(j1, j0 + (uint32_t)CM_HB * (uint32_t)__shfl_sync(0xFFFFFFFFu, bb, 0));
        };
        uint32_t jb = grab();                          // current block [jb, je)
        uint32_t je = min(j1, jb + CM_HB);
        uint32_t jb_next = jb < j1 ? grab() : j1;      // next block's first hash
        uint32_t j = jb;
        uint4 pre[2 * TW];                             // T0 draws = 2 * TW x 16 B per lane
        if (j < j1) {
            const uint4 *t4 = reinterpret_cast<const uint4 *>(p.table + (int64_t)j * T0 * TW);
#pragma unroll
            for (int i = 0; i < 2 * TW; i++) pre[i] = __ldg(t4 + 32 * i + lane);
        }
        while (j < j1) {
            __syncwarp();
#pragma unroll
            for (int i = 0; i < 2 * TW; i++) reinterpret_cast<uint4 *>(sbuf)[32 * i + lane] = pre[i];
            __syncwarp();
            const uint32_t jn = j + 1 < je ? j + 1 : jb_next;
            uint16_t *hres = hres_blk + (j - jb) * R;
            if (jn < j1) {
                const uint4 *t4 = reinterpret_cast<const uint4 *>(p.table + (int64_t)jn * T0 * TW);
#pragma unroll
                for (int i = 0; i < 2 * TW; i++) pre[i] = __ldg(t4 + 32 * i + lane);
            }
            const uint64_t keyj = p.S ^ ((uint64_t)j << 32);

            // ---- SWAR rounds (draws 0..32*NR0-1): lane = (4-row word, part); four
            //      packed draws per 16-byte shared load, B = nb in every byte, K = B & 0x7F
            const int w = lane % NWD, part = lane / NWD;
            uint32_t h4 = 0xFFFFFFFFu;                 // per byte: first green draw within the part
            {
                const uint4 *e4 = reinterpret_cast<const uint4 *>(sbuf + part * PD * TW);
                const uint8_t *xw = xs + 4 * w;
                constexpr int PER = 4 / TW;            // draws per 16-byte load
#pragma unroll
                for (int i4 = PD / PER - 1; i4 >= 0; i4--) {
                    const uint4 q4 = e4[i4];
                    const uint32_t w4[4] = {q4.x, q4.y, q4.z, q4.w};
#pragma unroll
                    for (int u = PER - 1; u >= 0; u--) {
                        uint32_t col, B;
                        if (TW == 1) {
                            col = w4[u] >> 8;
                            B = prmt(w4[u], 0u, 0x0000);                        // nb in every byte
                        } else {
                            col = w4[2 * u];
                            B = w4[2 * u + 1];
                        }
                        const uint32_t a = *reinterpret_cast<const uint32_t *>(xw + col);
                        const uint32_t s = (a & 0x7F7F7F7Fu) + (B & 0x7F7F7F7Fu);
                        const uint32_t g = (a & B) | (a & s) | (B & s);          // carry out of bit 7 (MAJ)
                        const uint32_t m = prmt(g, 0u, 0xBA98);                 // msb -> whole byte
                        h4 = (h4 & ~m) | ((uint32_t)(part * PD + PER * i4 + u) * 0x01010101u & m);
                    }
                }
            }
            if (P > 1) {                                // first part with a green wins, per byte
                spart[lane] = h4;
                __syncwarp();
                if (lane < NWD) {
                    uint32_t hw = 0xFFFFFFFFu;
#pragma unroll
                    for (int q2 = P - 1; q2 >= 0; q2--) {
                        const uint32_t o = spart[q2 * NWD + lane];
                        const uint32_t m = prmt(~o, 0u, 0xBA98);            // bytes of o that are green (< 0x80)
                        hw = (hw & ~m) | (o & m);
                    }
                    h4 = hw;
                }
                __syncwarp();
            }
            // ---- round-0 results -> hres, pending rows -> own1 --------------------
            int npend = 0;
            {
                const bool wl = lane < NWD;
                const uint32_t live4 = wl ? (uint32_t)sflag4[w] : 0u;
                // bytes: first green index (0..32*NR0-1) -> h = index + 1; 0xFF -> 0 (pending)
                const uint32_t v = ((h4 & 0x7F7F7F7Fu) + 0x01010101u) & 0x7F7F7F7Fu;
                if (wl) {
                    const uint32_t lo = prmt(v, 0u, 0x4140), hi = prmt(v, 0u, 0x4342);
                    // dead rows (all-zero) never turn green: h = cap
                    uint32_t l2 = lo, h2 = hi;
                    if (!(live4 & 1u)) l2 = (l2 & 0xFFFF0000u) | p.cap;
                    if (!(live4 & 2u)) l2 = (l2 & 0x0000FFFFu) | (p.cap << 16);
                    if (!(live4 & 4u)) h2 = (h2 & 0xFFFF0000u) | p.cap;
                    if (!(live4 & 8u)) h2 = (h2 & 0x0000FFFFu) | (p.cap << 16);
                    *reinterpret_cast<uint2 *>(hres + 4 * w) = make_uint2(l2, h2);
                    const uint32_t valid4 = (4 * w + 4 <= nr) ? 0xFu : ((1u << max(0, nr - 4 * w)) - 1u);
                    sat += __popc(valid4 & ~live4);
                }
#pragma unroll
                for (int b = 0; b < 4; b++) {
                    const int row = 4 * w + b;
                    const bool pend = wl && row < nr && ((live4 >> b) & 1u) && ((v >> (8 * b)) & 0xFFu) == 0u;
                    const unsigned pm = __ballot_sync(0xFFFFFFFFu, pend);
                    if (pend) own1[npend + __popc(pm & ((1u << lane) - 1))] = (uint16_t)row;
                    npend += __popc(pm);
                }
            }
            __syncwarp();
            const uint16_t *cur = own1;
            uint32_t q = NR0;
            switch (C) {
                case 8: npend = cm_rounds<8, TW>(p, sbuf, swin, xs, keyj, hres, cur, own0, own1, npend, &q); break;
                case 16: npend = cm_rounds<16, TW>(p, sbuf, swin, xs, keyj, hres, cur, own0, own1, npend, &q); break;
                default: npend = cm_rounds<32, TW>(p, sbuf, swin, xs, keyj, hres, cur, own0, own1, npend, &q); break;
            }
            if (npend > 0 && q * 32 >= p.cap) {        // a9: no green draw before the cap
                for (int i = lane; i < npend; i += 32) {
                    hres[cur[i]] = (uint16_t)p.cap;
                    sat++;
                }
                npend = 0;
            }
            if (npend > 0) {                           // draw-parallel stragglers (<= CM_STRAG)
                int rr[CM_STRAG];
                unsigned live = 0;
#pragma unroll
                for (int i = 0; i < CM_STRAG; i++) {
                    rr[i] = i < npend ? (int)cur[i] : 0;
                    if (i < npend) live |= 1u << i;
                }
                for (; live && q * 32 < p.cap; q++) {
                    const uint32_t t = q * 32 + lane;
                    uint2 dd;
                    if (t < (uint32_t)T0) dd = cm_get<TW>(sbuf, t);
                    else {
                        const uint32_t pw = cm_late(p, keyj, t);
                        dd = make_uint2(pw >> 8, (pw & 0xFFu) ^ 0xFFu);
                    }
                    const uint32_t off = dd.y, dcol = dd.x;
#pragma unroll
                    for (int i = 0; i < CM_STRAG; i++) {
                        if (live & (1u << i)) {
                            const uint32_t xv = xs[dcol + rr[i]];
                            const unsigned gm = __ballot_sync(0xFFFFFFFFu, xv > off);
                            if (gm) {
                                if (lane == 0) hres[rr[i]] = (uint16_t)(q * 32 + __ffs(gm));
                                live &= ~(1u << i);
                            }
                        }
                    }
                }
#pragma unroll
                for (int i = 0; i < CM_STRAG; i++)
                    if ((live & (1u << i)) && lane == 0) {
                        hres[rr[i]] = (uint16_t)p.cap;
                        sat++;
                    }
            }
            __syncwarp();
            if (j + 1 == je) {
                // ---- a9: flush the block: row r's hashes jb..je-1 are contiguous in
                //      sig, one 4-hash store per row when the block is full and aligned
                __syncwarp();
                using sig_t = typename std::conditional<SIGB == 1, uint8_t, uint16_t>::type;
                sig_t *ptr = reinterpret_cast<sig_t *>(p.sig) + (row0 + lane) * (int64_t)p.k + jb;
                const int64_t step = 32 * (int64_t)p.k;
                const int nh = (int)(je - jb);
                if (nh == CM_HB && p.vec_flush) {
                    for (int r = lane; r < nr; r += 32, ptr += step) {
                        uint32_t hv[CM_HB];
#pragma unroll
                        for (int u = 0; u < CM_HB; u++) hv[u] = hres_blk[u * R + r];
                        if (SIGB == 2) {
                            const uint4 v = make_uint4(hv[0] | (hv[1] << 16), hv[2] | (hv[3] << 16),
                                                       hv[4] | (hv[5] << 16), hv[6] | (hv[7] << 16));
                            if (p.vec_flush == 2) {
                                *reinterpret_cast<uint4 *>(ptr) = v;               // 16-byte aligned rows
                            } else {
                                reinterpret_cast<uint2 *>(ptr)[0] = make_uint2(v.x, v.y);
                                reinterpret_cast<uint2 *>(ptr)[1] = make_uint2(v.z, v.w);
                            }
                        } else {
                            *reinterpret_cast<uint2 *>(ptr) = make_uint2(hv[0] | (hv[1] << 8) | (hv[2] << 16) | (hv[3] << 24),
                                                                         hv[4] | (hv[5] << 8) | (hv[6] << 16) | (hv[7] << 24));
                        }
                    }
                } else {
                    for (int r = lane; r < nr; r += 32, ptr += step)
                        for (int u = 0; u < nh; u++) ptr[u] = (sig_t)hres_blk[u * R + r];
                }
                jb = jb_next;
                je = min(j1, jb + CM_HB);
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

static size_t cm_smem(int D, int R, int Rp, int TW) {
    return (((size_t)D * Rp + 15) & ~(size_t)15) + (size_t)CM_NW * (T0 + 32) * 4 * TW +
           (size_t)CM_NW * 32 * 4 + (size_t)CM_NW * CM_HB * R * 2 + (size_t)CM_NW * 2 * R * 2 + (size_t)(R / 4) + 16;
}

template <int SIGB, int P, int TW>
static void cm_launch(const CmParams &p, size_t smem, int grid, cudaStream_t s) {
    // SWAR rounds before the pending-list rounds: measured best 1 for the
    // 128-row tile (c2: 0.609 vs 0.630 ms) and 2 for the 32-row tile (c5:
    // 5.39 vs 6.41 ms per 262,144 rows); WMH_CM_SWAR_ROUNDS overrides
    static const int env_nr0 = getenv("WMH_CM_SWAR_ROUNDS") ? atoi(getenv("WMH_CM_SWAR_ROUNDS")) : 0;
    const int nr0 = env_nr0 == 1 || env_nr0 == 2 ? env_nr0 : (P == 1 ? 1 : 2);
    auto kern = nr0 == 1 ? hash_tiled_cm_kernel<SIGB, P, 1, TW> : hash_tiled_cm_kernel<SIGB, P, 2, TW>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kernel_timer_begin(s);
    kern<<<grid, CM_NT, smem, s>>>(p);
    kernel_timer_end(s);
}

// does the column-major byte tile hold its full 128 rows for these rows?
bool tiled_cm_full_tile(const HashArgs &a) {
    int dev = 0;
    cudaGetDevice(&dev);
    int smem_optin = 0;
    cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    return cm_smem((int)a.rows.dim, 128, 132, 1) <= (size_t)smem_optin;
}

wmh_status launch_hash_tiled_cm(const HashArgs &a, bool *handled) {
    *handled = false;
    const int D = (int)a.rows.dim;
    if (a.rows.kind != WMH_DENSE || (D & 3) || ((uintptr_t)a.rows.dense & 3)) return WMH_OK;
    int dev = 0;
    cudaGetDevice(&dev);
    int smem_optin = 0;
    cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    // rows per tile R = 128 / P; column stride Rp = R + 4 (Rp/4 odd: draw-
    // parallel accesses to random columns spread over the banks)
    // draw-table words per draw: 1 (packed; measured: c2 0.612 vs 0.623 ms with
    // 2 words, c5 slice 5.41 vs 5.82 ms); WMH_CM_TW=2 selects the (c*Rp, B) pairs
    static const int tw_env = getenv("WMH_CM_TW") ? atoi(getenv("WMH_CM_TW")) : 0;
    int P = 1, R = 0, Rp = 0, TW = 1;
    for (; P <= 4; P *= 2) {
        R = 128 / P;
        Rp = R + 4;
        TW = tw_env == 2 ? 2 : 1;
        if (cm_smem(D, R, Rp, TW) <= (size_t)smem_optin) break;
    }
    if (P > 4) return WMH_OK;
    const size_t smem = cm_smem(D, R, Rp, TW);
    *handled = true;

    const int64_t n_tiles = (a.rows.n_rows + R - 1) / R;
    const int sms = num_sms();
    // >= 8 items per SM for balance, but >= WMH_MIN_HCHUNK hashes per item: each
    // item stages its whole tile, so small batches must not slice k too thin
    // (a 3,300-row batch of c2 in 16-hash items ran 3x slower than its share)
    static const int min_hc = getenv("WMH_MIN_HCHUNK") ? std::max(8, atoi(getenv("WMH_MIN_HCHUNK"))) : 128;
    int n_hchunks = (int)max((int64_t)1, min((int64_t)(a.k + min_hc - 1) / min_hc, ((int64_t)sms * 8 + n_tiles - 1) / n_tiles));
    static const int hc_env = getenv("WMH_CM_HCHUNKS") ? atoi(getenv("WMH_CM_HCHUNKS")) : 0;
    if (hc_env > 0) n_hchunks = (int)min((int64_t)hc_env, (int64_t)(a.k + CM_HB - 1) / CM_HB);
    const int hchunk = (int)(((a.k + n_hchunks - 1) / n_hchunks + CM_HB - 1) / CM_HB * CM_HB);   // blocks stay 4-aligned
    n_hchunks = (int)((a.k + hchunk - 1) / hchunk);

    uint8_t *scratch = nullptr;
    const size_t tab_bytes = (size_t)a.k * T0 * sizeof(uint32_t) * TW;
    WMH_CUDA_TRY(cudaMallocAsync((void **)&scratch, tab_bytes + 256, a.stream), "tiled scratch alloc");
    uint32_t *table = reinterpret_cast<uint32_t *>(scratch);
    unsigned long long *ctr = reinterpret_cast<unsigned long long *>(scratch + tab_bytes);
    WMH_CUDA_TRY(cudaMemsetAsync(ctr, 0, sizeof(unsigned long long), a.stream), "tiled counter memset");
    const uint32_t uni_m = (a.L->flags & WMH_LAYOUT_UNIFORM) ? a.L->uniform_m : 0u;
    const uint32_t M = (uint32_t)a.L->M;
    {
        const int64_t total = (int64_t)a.k * T0;
        const int blocks = (int)min((int64_t)num_sms() * 8, (total + 255) / 256);
        if (TW == 2) cm_table_kernel<2><<<blocks, 256, 0, a.stream>>>(table, a.k, a.S, M, a.L->cell_pack, uni_m, (uint32_t)Rp, a.cap);
        else cm_table_kernel<1><<<blocks, 256, 0, a.stream>>>(table, a.k, a.S, M, a.L->cell_pack, uni_m, (uint32_t)Rp, a.cap);
        count_launch();
        if (cudaGetLastError() != cudaSuccess) { cudaFreeAsync(scratch, a.stream); return cuda_fail(cudaGetLastError(), "cm table launch"); }
    }

    CmParams p;
    p.x = a.rows.dense;
    p.n_rows = a.rows.n_rows;
    p.D = D;
    p.R = R;
    p.Rp = Rp;
    p.n_hchunks = n_hchunks;
    p.hchunk = hchunk;
    p.n_items = n_tiles * n_hchunks;
    p.k = a.k;
    p.cap = a.cap;
    p.M = M;
    p.uni_m = uni_m;
    p.S = a.S;
    p.chunk = a.chunk == 4 ? 8 : a.chunk;
    // vectorised block flush: 1 = 8-byte stores (k % 4 == 0, sig 8-aligned), 2 = one 16-byte
    // store per row (uint16 rows 16-byte aligned: k % 8 == 0, sig 16-aligned); uint8 rows: 8 bytes
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
#define WMH_CM_GO(SB)                                                        \
    do {                                                                     \
        if (TW == 2) {                                                       \
            if (P == 1) cm_launch<SB, 1, 2>(p, smem, grid, a.stream);        \
            else if (P == 2) cm_launch<SB, 2, 2>(p, smem, grid, a.stream);   \
            else cm_launch<SB, 4, 2>(p, smem, grid, a.stream);               \
        } else {                                                             \
            if (P == 1) cm_launch<SB, 1, 1>(p, smem, grid, a.stream);        \
            else if (P == 2) cm_launch<SB, 2, 1>(p, smem, grid, a.stream);   \
            else cm_launch<SB, 4, 1>(p, smem, grid, a.stream);               \
        }                                                                    \
    } while (0)
    if (a.sig_bytes == 1) WMH_CM_GO(1);
    else WMH_CM_GO(2);
#undef WMH_CM_GO
    WMH_LAUNCH_CHECK("hash_tiled_cm launch");
    if (getenv("WMH_TILED_STATS"))
        fprintf(stderr, "[wmh tiled cm] R=%d Rp=%d P=%d TW=%d grid=%d items=%lld hchunk=%d smem=%zu\n", R, Rp, P, TW,
                grid, (long long)p.n_items, hchunk, smem);
    cudaFreeAsync(scratch, a.stream);
    return WMH_OK;
}

}  // namespace wmh
