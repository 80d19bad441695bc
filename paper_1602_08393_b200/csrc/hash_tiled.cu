// hash_tiled.cu -- WMH_ALGO_TILED for dense rows: the B200 form of Alg. 3.
//
// The paper's draw stream is independent of x ("consistency", P:190-191:
// every vector sees the same r_1, r_2, ... for a given hash), so one draw
// r_t of hash j can be tested against MANY rows.  A CTA stages a tile of R
// rows in shared memory; a warp takes one hash j at a time and walks the
// stream: the first T0 = 256 draws of every hash come from a per-launch table
// (prefetched one hash ahead into a per-warp shared buffer), later ones are
// computed on the fly (a6).  Draws are broadcast into every lane's registers
// and each lane tests them against the rows it owns (lane = row): green iff
// x[row][c_t] > off_t (Alg. 5).  A row is tested against C draws
// (C = 4..32, picked per tile from its effective sparsity s = |x|_1 / M,
// Eq. 17) before it is re-queued: the first green t gives h = t + 1
// (Alg. 3 / Def.), rows without one stay on the warp's pending
// list.  When few rows remain pending the warp switches to draw-parallel
// mode (lane = draw, loop over the pending rows, ballot + ffs finds the first
// green).  Rows still pending at the cap get h = cap (reading R9).
//
// Shared-memory rows use an odd word stride, so the 32 lanes of a
// row-parallel test (same c_t, 32 different rows) hit 32 different banks.
#include <stdio.h>
#include <stdlib.h>

#include "common.cuh"

namespace wmh {

constexpr int STRAG_MAX = 4;            // max pending rows handled draw-parallel (threshold: p.strag)

// table[j * T0 + t] = (c * cmul, r_t - CompToM[c]) of draw r_t of hash j, t < T0
// (cmul = 1 for row-major tiles, the column stride for column-major ones).
__global__ void draw_table_kernel(uint2 *__restrict__ table, uint32_t k, uint64_t S, uint32_t M,
                                  const uint32_t *__restrict__ pack, uint32_t uni_m, uint32_t cmul,
                                  const uint32_t *__restrict__ i2c, const uint32_t *__restrict__ c2m) {
    const int64_t total = (int64_t)k * T0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        uint32_t j = (uint32_t)(i / T0), t = (uint32_t)(i % T0);
        const uint2 d = cell_lookup(draw_r(S, j, t, M), pack, uni_m, i2c, c2m);
        table[i] = make_uint2(d.x * cmul, d.y);
    }
}

wmh_status launch_draw_table(uint2 *table, uint32_t k, uint64_t S, uint32_t M, const uint32_t *pack, uint32_t uni_m,
                             uint32_t cmul, cudaStream_t s, const uint32_t *i2c, const uint32_t *c2m) {
    const int64_t total = (int64_t)k * T0;
    const int blocks = (int)min((int64_t)num_sms() * 8, (total + 255) / 256);
    draw_table_kernel<<<blocks, 256, 0, s>>>(table, k, S, M, pack, uni_m, cmul, i2c, c2m);
    WMH_LAUNCH_CHECK("draw table launch");
    return WMH_OK;
}

struct TiledParams {
    const uint8_t *x;
    int64_t n_rows;
    int D, SW, R;               // dim, smem row stride (words, odd), rows per tile
    int n_hchunks, hchunk;      // hash chunks per tile item
    int64_t n_items;
    uint32_t k, cap, M, uni_m;
    uint64_t S;
    int chunk;                  // 0 = auto
    int strag;                  // pending rows at or below which a warp goes draw-parallel
    const uint2 *table;         // [k][T0] (c, off)
    const uint32_t *pack;
    void *sig;
    unsigned long long *n_sat;
    unsigned long long *item_ctr;
    unsigned long long *stats;  // debug (WMH_TILED_STATS=1): tiles per C, sum of tile s * 1e9
};

template <int SIGB>
__device__ __forceinline__ void store_sig(void *sig, int64_t idx, uint32_t h) {
    if (SIGB == 1) reinterpret_cast<uint8_t *>(sig)[idx] = (uint8_t)h;
    else reinterpret_cast<uint16_t *>(sig)[idx] = (uint16_t)h;
}

// (c, off) of draw t >= T0 of hash j (computed: a6 + Alg. 5 lookup).
__device__ __forceinline__ uint2 late_cell(const TiledParams &p, uint64_t keyj, uint32_t t) {
    return unpack_cell(cell_of(mulhi_range(splitmix64(keyj ^ (uint64_t)t), p.M), p.pack, p.uni_m));
}

// Per-warp state of the hash being processed.
struct HashCtx {
    const uint2 *buf;           // shared: (c, off) of draws 0..T0-1 of hash j
    uint2 *win;                 // shared: 32-draw window for draws >= T0
    uint32_t j;
    uint64_t keyj;
    int64_t row0;
};

// Row-parallel rounds over the warp's pending list (cur), C draws per
// re-queue.  Returns the number of rows still pending (left in cur) and the
// next round in *q; stops when <= p.strag rows remain or at the cap.
template <int SIGB, int C>
__device__ __forceinline__ int rounds_row_parallel(const TiledParams &p, const HashCtx &hx, const uint8_t *srow_bytes,
                                                   int SW4, const uint16_t *&cur, uint16_t *own0, uint16_t *own1,
                                                   int npend, uint32_t *q_io) {
    const int lane = threadIdx.x & 31;
    uint32_t q = *q_io;
    int flip = 0;
    while (npend > p.strag && q * 32 < p.cap) {
        const uint2 *src;
        if (q * 32 < (uint32_t)T0) {
            src = hx.buf + q * 32;
        } else {                                             // beyond the table: compute this round
            const uint2 c = late_cell(p, hx.keyj, q * 32 + lane);
            __syncwarp();
            hx.win[lane] = c;
            __syncwarp();
            src = hx.win;
        }
        const bool cap_round = q * 32 + 32 > p.cap;
#pragma unroll
        for (int sub = 0; sub < 32 / C; sub++) {
            if (npend == 0) break;
            uint32_t dc[C], doff[C];
#pragma unroll
            for (int i = 0; i < C / 2; i++) {
                const uint4 v = reinterpret_cast<const uint4 *>(src + sub * C)[i];
                dc[2 * i] = v.x; doff[2 * i] = v.y; dc[2 * i + 1] = v.z; doff[2 * i + 1] = v.w;
            }
            if (cap_round) {                                 // draws at or past the cap never turn green
#pragma unroll
                for (int tt = 0; tt < C; tt++)
                    if (q * 32 + sub * C + tt >= p.cap) doff[tt] = 0xFFFFFFFFu;
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
                    // first green among the C draws: NCH independent select
                    // chains over interleaved draws (ILP), combined by min.
                    constexpr int NCH = C >= 16 ? 4 : 2;
                    const uint8_t *row = srow_bytes + r * SW4;
                    uint32_t hc[NCH];
#pragma unroll
                    for (int c = 0; c < NCH; c++) hc[c] = C;
#pragma unroll
                    for (int tt = C - 1; tt >= 0; tt--) {
                        const uint32_t v = row[dc[tt]];
                        hc[tt % NCH] = (v > doff[tt]) ? (uint32_t)tt : hc[tt % NCH];
                    }
                    h = hc[0];
#pragma unroll
                    for (int c = 1; c < NCH; c++) h = min(h, hc[c]);
                }
                const bool still = active && h == C;
                if (active && !still)
                    store_sig<SIGB>(p.sig, (hx.row0 + r) * (int64_t)p.k + hx.j, q * 32 + sub * C + h + 1);
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

template <int SIGB, int NT>
__global__ void __launch_bounds__(NT, (NT == 256 ? 2 : 1)) hash_tiled_dense_kernel(const TiledParams p) {
    constexpr int NW = NT / 32;
    extern __shared__ __align__(16) uint32_t smem[];
    const int R = p.R, SW = p.SW, SW4 = p.SW * 4;
    uint32_t *srows = smem;                                             // [R][SW] words
    uint2 *sbuf_all = reinterpret_cast<uint2 *>(smem + R * SW);         // [NW][T0] draws (c, off)
    uint2 *swin_all = sbuf_all + NW * T0;                               // [NW][32] late draws
    uint16_t *spend_all = reinterpret_cast<uint16_t *>(swin_all + NW * 32);   // [NW][2][R]
    uint16_t *salive = spend_all + NW * 2 * R;                          // [R] alive row list
    uint8_t *sflag = reinterpret_cast<uint8_t *>(salive + R);           // [R] row has |x|_1 > 0
    __shared__ long long s_item, s_next;
    __shared__ int s_hash, s_nalive;
    __shared__ unsigned long long s_xsum;

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint2 *sbuf = sbuf_all + warp * T0;
    uint2 *swin = swin_all + warp * 32;
    uint16_t *own0 = spend_all + warp * 2 * R, *own1 = own0 + R;
    const uint8_t *srow_bytes = reinterpret_cast<const uint8_t *>(srows);
    unsigned long long sat = 0;
    const bool vec16 = (p.D % 16 == 0) && ((reinterpret_cast<uintptr_t>(p.x) & 15) == 0);
    if (threadIdx.x == 0) s_next = (long long)atomicAdd(p.item_ctr, 1ull);

    for (;;) {
        __syncthreads();                                    // previous item fully done with smem
        if (threadIdx.x == 0) {
            s_item = s_next;                                // claimed one item ahead
            s_next = (long long)atomicAdd(p.item_ctr, 1ull);
            s_hash = 0;
            s_xsum = 0;
            s_nalive = 0;
        }
        __syncthreads();
        const long long item = s_item;
        if (item >= p.n_items) break;
        if (s_next < p.n_items) {                           // warm L2 with the next item's rows
            const int64_t nrow0 = (s_next / p.n_hchunks) * R;
            const int64_t nbytes = min((int64_t)R, p.n_rows - nrow0) * (int64_t)p.D;
            const char *base = reinterpret_cast<const char *>(p.x + nrow0 * (int64_t)p.D);
            for (int64_t off = (int64_t)threadIdx.x * 128; off < nbytes; off += (int64_t)NT * 128)
                asm volatile("prefetch.global.L2 [%0];" ::"l"(base + off));
        }
        const int64_t tile = item / p.n_hchunks;
        const int hc = (int)(item % p.n_hchunks);
        const int64_t row0 = tile * R;
        const int nr = (int)min((int64_t)R, p.n_rows - row0);
        const uint32_t j0 = (uint32_t)hc * p.hchunk;
        const uint32_t j1 = min(p.k, j0 + (uint32_t)p.hchunk);

        // ---- a5: stage the tile (one warp per row, 16-byte loads), |x|_1 per row ----
        for (int r = warp; r < nr; r += NW) {
            const uint8_t *g = p.x + (row0 + r) * (int64_t)p.D;
            uint32_t *srow = srows + r * SW;
            uint32_t acc = 0;
            if (vec16) {
                for (int c = lane; c < p.D / 16; c += 32) {
                    const uint4 v = __ldg(reinterpret_cast<const uint4 *>(g) + c);
                    srow[4 * c + 0] = v.x; srow[4 * c + 1] = v.y; srow[4 * c + 2] = v.z; srow[4 * c + 3] = v.w;
                    acc = __dp4a(v.x, 0x01010101u, acc);
                    acc = __dp4a(v.y, 0x01010101u, acc);
                    acc = __dp4a(v.z, 0x01010101u, acc);
                    acc = __dp4a(v.w, 0x01010101u, acc);
                }
            } else {
                uint8_t *sb = reinterpret_cast<uint8_t *>(srow);
                for (int c = lane; c < p.D; c += 32) {
                    const uint8_t v = __ldg(g + c);
                    sb[c] = v;
                    acc += v;
                }
            }
            for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xFFFFFFFFu, acc, o);
            if (lane == 0 && acc) atomicAdd(&s_xsum, (unsigned long long)acc);
            // alive flag, compacted below; an all-zero row never turns green (h = cap)
            if (lane == 0) sflag[r] = acc != 0;
        }
        __syncthreads();
        // compact the alive rows into salive (warp 0); dead rows are rare
        if (warp == 0) {
            int n = 0;
            for (int base = 0; base < nr; base += 32) {
                const int r = base + lane;
                const bool alive = r < nr && sflag[r];
                const unsigned m = __ballot_sync(0xFFFFFFFFu, alive);
                if (alive) salive[n + __popc(m & ((1u << lane) - 1))] = (uint16_t)r;
                n += __popc(m);
            }
            if (lane == 0) s_nalive = n;
        }
        __syncthreads();
        const int nalive = s_nalive;
        int C = p.chunk;
        if (C == 0) {                   // C from the tile's effective sparsity
            const double s = nalive ? (double)s_xsum / ((double)nalive * (double)p.M) : 1.0;
            C = s > 0.2 ? 8 : s > 0.1 ? 16 : 32;
            if (p.stats && threadIdx.x == 0) atomicAdd(p.stats + 5, (unsigned long long)(s * 1e9));
        }
        if (p.stats && threadIdx.x == 0) atomicAdd(p.stats + (31 - __clz(C)) - 2, 1ull);

        // ---- hashes of this item: one warp per hash, dynamically assigned, the
        //      next hash's table prefetched while the current one runs ------------
        auto grab = [&]() {
            int jj = 0;
            if (lane == 0) jj = atomicAdd(&s_hash, 1);
            return j0 + (uint32_t)__shfl_sync(0xFFFFFFFFu, jj, 0);
        };
        uint32_t j = grab();
        uint4 pre[4];                                      // this lane's 8 draws of the next hash
        if (j < j1) {
            const uint4 *t4 = reinterpret_cast<const uint4 *>(p.table + (int64_t)j * T0);
#pragma unroll
            for (int i = 0; i < 4; i++) pre[i] = __ldg(t4 + 32 * i + lane);
        }
        while (j < j1) {
            __syncwarp();
#pragma unroll
            for (int i = 0; i < 4; i++) reinterpret_cast<uint4 *>(sbuf)[32 * i + lane] = pre[i];
            __syncwarp();
            const uint32_t jn = grab();
            if (jn < j1) {
                const uint4 *t4 = reinterpret_cast<const uint4 *>(p.table + (int64_t)jn * T0);
#pragma unroll
                for (int i = 0; i < 4; i++) pre[i] = __ldg(t4 + 32 * i + lane);
            }
            HashCtx hx;
            hx.buf = sbuf;
            hx.win = swin;
            hx.j = j;
            hx.keyj = p.S ^ ((uint64_t)j << 32);
            hx.row0 = row0;
            const uint16_t *cur = salive;
            int npend = nalive;
            uint32_t q = 0;
            switch (C) {
                case 4: npend = rounds_row_parallel<SIGB, 4>(p, hx, srow_bytes, SW4, cur, own0, own1, npend, &q); break;
                case 8: npend = rounds_row_parallel<SIGB, 8>(p, hx, srow_bytes, SW4, cur, own0, own1, npend, &q); break;
                case 16: npend = rounds_row_parallel<SIGB, 16>(p, hx, srow_bytes, SW4, cur, own0, own1, npend, &q); break;
                default: npend = rounds_row_parallel<SIGB, 32>(p, hx, srow_bytes, SW4, cur, own0, own1, npend, &q); break;
            }
            // ---- a9: rows with no green draw before the cap saturate ----------
            if (npend > 0 && q * 32 >= p.cap) {
                for (int i = lane; i < npend; i += 32) {
                    store_sig<SIGB>(p.sig, (row0 + cur[i]) * (int64_t)p.k + j, p.cap);
                    sat++;
                }
                npend = 0;
            }
            // ---- draw-parallel mode for the last <= p.strag rows ------------------
            if (npend > 0) {
                int rr[STRAG_MAX];
                unsigned live = 0;
#pragma unroll
                for (int i = 0; i < STRAG_MAX; i++) {
                    rr[i] = i < npend ? (int)cur[i] : 0;
                    if (i < npend) live |= 1u << i;
                }
                for (; live && q * 32 < p.cap; q++) {
                    const uint32_t t = q * 32 + lane;
                    const uint2 cell = t < (uint32_t)T0 ? sbuf[t] : late_cell(p, hx.keyj, t);
                    const uint32_t c = cell.x, off = t < p.cap ? cell.y : 0xFFFFFFFFu;
#pragma unroll
                    for (int i = 0; i < STRAG_MAX; i++) {
                        if (live & (1u << i)) {
                            const uint32_t v = srow_bytes[rr[i] * SW4 + c];
                            const unsigned g = __ballot_sync(0xFFFFFFFFu, v > off);
                            if (g) {
                                if (lane == 0)
                                    store_sig<SIGB>(p.sig, (row0 + rr[i]) * (int64_t)p.k + j, q * 32 + __ffs(g));
                                live &= ~(1u << i);
                            }
                        }
                    }
                }
#pragma unroll
                for (int i = 0; i < STRAG_MAX; i++)
                    if ((live & (1u << i)) && lane == 0) {
                        store_sig<SIGB>(p.sig, (row0 + rr[i]) * (int64_t)p.k + j, p.cap);
                        sat++;
                    }
            }
            j = jn;
        }
        // all-zero rows of the tile: h = cap for every hash of the item (reading R12)
        if (nalive < nr) {
            __syncthreads();
            for (int r = warp; r < nr; r += NW) {
                if (sflag[r]) continue;
                for (uint32_t jj = j0 + lane; jj < j1; jj += 32) {
                    store_sig<SIGB>(p.sig, (row0 + r) * (int64_t)p.k + jj, p.cap);
                    sat++;
                }
            }
        }
    }
    if (p.n_sat) {
        for (int o = 16; o; o >>= 1) sat += __shfl_xor_sync(0xFFFFFFFFu, sat, o);
        if (lane == 0 && sat) atomicAdd(p.n_sat, sat);
    }
}

static size_t tiled_smem(int R, int SW, int NW) {
    return (size_t)R * SW * 4 + (size_t)NW * (T0 + 32) * 8 + (size_t)NW * 2 * R * 2 + (size_t)R * 3 + 16;
}

template <int SIGB, int NT>
static wmh_status launch_tiled(const TiledParams &p, size_t smem, int grid, cudaStream_t s) {
    auto *fn = hash_tiled_dense_kernel<SIGB, NT>;
    WMH_CUDA_TRY(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem), "tiled smem attr");
    kernel_timer_begin(s);
    fn<<<grid, NT, smem, s>>>(p);
    kernel_timer_end(s);
    WMH_LAUNCH_CHECK("hash_tiled_dense launch");
    return WMH_OK;
}

wmh_status launch_hash_tiled(const HashArgs &a, bool *handled) {
    *handled = false;
    // the tiles test uint8 weights against 8-bit cell offsets: narrow layouts only
    if ((a.L->flags & WMH_LAYOUT_WIDE) || weight_bytes(a.rows) != 1) return WMH_OK;
    // sparse rows are hashed by the INDEX kernel (or SIMPLE); the tiles test dense rows
    if (a.rows.kind != WMH_DENSE) return WMH_OK;
    // column-major tile with the SIMD first round (hash_tiled_cm.cu) unless
    // WMH_TILED_RM=1 selects this row-major kernel
    static const bool force_rm = getenv("WMH_TILED_RM") != nullptr;
    // bit-plane tile (hash_tiled_bs.cu) for long rows -- where the byte tile
    // would hold fewer than 128 rows and the planes of >= 2 groups fit
    // (measured: c5's recipe, 10^6 rows, NB = 6: 18.1 vs 21.2 ms; on c2's
    // 128-row tile the SWAR byte tile stays ahead, 0.58 vs 0.75 ms);
    // WMH_TILED_BS=1 / 0 or the WMH_OPT_TILE_* flags force the choice
    // the lane-per-draw bit-sliced tile (hash_bitslice.cu) for long rows, where
    // the byte tile would hold fewer than 128 rows (c5, D = 4096: 12.4 ms per
    // 2^20 rows vs 17.95 for the round-1 bit-plane tile and 21 for the byte
    // tile); on c2's 128-row byte tile the SWAR byte test stays ahead (0.58 vs
    // 1.03 ms).  WMH_OPT_TILE_BITSLICE forces it; WMH_TILED_BV=0 drops it from AUTO
    static const int bv_env = getenv("WMH_TILED_BV") ? atoi(getenv("WMH_TILED_BV")) : -1;
    if (!force_rm && (a.tile == 3 || (a.tile == 0 && bv_env != 0 && (bv_env == 1 || !tiled_cm_full_tile(a))))) {
        const wmh_status vst = launch_hash_bitslice(a, handled);
        if (*handled && a.tile_used) *a.tile_used = 3;
        if (vst != WMH_OK || *handled) return vst;
    }
    static const int bs_env = getenv("WMH_TILED_BS") ? atoi(getenv("WMH_TILED_BS")) : -1;
    const bool want_bs = a.tile == 2 || (a.tile == 0 && (bs_env == 1 || (bs_env != 0 && !tiled_cm_full_tile(a))));
    if (!force_rm && want_bs) {
        const wmh_status bst = launch_hash_tiled_bs(a, handled);
        if (*handled && a.tile_used) *a.tile_used = 2;
        if (bst != WMH_OK || *handled) return bst;
    }
    if (!force_rm) {
        const wmh_status cst = launch_hash_tiled_cm(a, handled);
        if (*handled && a.tile_used) *a.tile_used = 1;
        if (cst != WMH_OK || *handled) return cst;
    }
    const int D = (int)a.rows.dim;
    const int SW = (((D + 3) >> 2) | 1);                  // odd word stride: conflict-free lane=row tests
    int dev = 0;
    cudaGetDevice(&dev);
    int smem_optin = 0, smem_sm = 0;
    cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
    static const int force_ctas = getenv("WMH_TILED_CTAS") ? atoi(getenv("WMH_TILED_CTAS")) : 0;
    // One 512-thread CTA per SM with the largest tile that fits (measured
    // faster than two 256-thread CTAs with half-size tiles); WMH_TILED_CTAS=2
    // selects the latter.
    int ctas = force_ctas == 2 ? 2 : 1, NT = 256, R = 0;
    for (; ctas >= 1; ctas--) {
        NT = ctas == 2 ? 256 : 512;
        size_t budget = min((size_t)smem_optin, (size_t)smem_sm / ctas - 1024);
        R = 256;
        while (R >= 32 && tiled_smem(R, SW, NT / 32) > budget) R -= 4;   // R % 4 == 0 keeps sbuf 16B-aligned
        if (R >= 32) break;
    }
    if (R < 32) return WMH_OK;                            // rows too long for a 32-row tile
    const size_t smem = tiled_smem(R, SW, NT / 32);
    *handled = true;

    const int64_t n_tiles = (a.rows.n_rows + R - 1) / R;
    const int sms = num_sms();
    // split the k hashes into chunks so there are >= ~8 items per resident CTA
    const int64_t slots = (int64_t)sms * ctas;
    int n_hchunks = (int)max((int64_t)1, min((int64_t)a.k / 8, (slots * 8 + n_tiles - 1) / n_tiles));
    n_hchunks = max(1, min(n_hchunks, (int)a.k));
    const int hchunk = (int)((a.k + n_hchunks - 1) / n_hchunks);
    n_hchunks = (int)((a.k + hchunk - 1) / hchunk);

    uint8_t *scratch = nullptr;
    const size_t tab_bytes = (size_t)a.k * T0 * sizeof(uint2);
    WMH_CUDA_TRY(cudaMallocAsync((void **)&scratch, tab_bytes + 256, a.stream), "tiled scratch alloc");
    uint2 *table = reinterpret_cast<uint2 *>(scratch);
    unsigned long long *ctr = reinterpret_cast<unsigned long long *>(scratch + tab_bytes);
    WMH_CUDA_TRY(cudaMemsetAsync(ctr, 0, 8 * sizeof(unsigned long long), a.stream), "tiled counter memset");
    static const bool want_stats = getenv("WMH_TILED_STATS") != nullptr;

    const uint32_t uni_m = (a.L->flags & WMH_LAYOUT_UNIFORM) ? a.L->uniform_m : 0u;
    const uint32_t M = (uint32_t)a.L->M;
    {
        const wmh_status tst = launch_draw_table(table, a.k, a.S, M, a.L->cell_pack, uni_m, 1u, a.stream);
        if (tst != WMH_OK) { cudaFreeAsync(scratch, a.stream); return tst; }
    }
    TiledParams p;
    p.x = a.rows.dense;
    p.n_rows = a.rows.n_rows;
    p.D = D;
    p.SW = SW;
    p.R = R;
    p.n_hchunks = n_hchunks;
    p.hchunk = hchunk;
    p.n_items = n_tiles * n_hchunks;
    p.k = a.k;
    p.cap = a.cap;
    p.M = M;
    p.uni_m = uni_m;
    p.S = a.S;
    p.chunk = a.chunk;
    static const int strag_env = getenv("WMH_TILED_STRAG") ? atoi(getenv("WMH_TILED_STRAG")) : -1;
    p.strag = strag_env >= 0 ? min(strag_env, STRAG_MAX) : 4;
    p.table = table;
    p.pack = a.L->cell_pack;
    p.sig = a.sig;
    p.n_sat = a.n_sat;
    p.item_ctr = ctr;
    p.stats = want_stats ? ctr + 1 : nullptr;
    const int grid = (int)min(slots, p.n_items);
    wmh_status st;
    if (a.sig_bytes == 1) st = NT == 256 ? launch_tiled<1, 256>(p, smem, grid, a.stream) : launch_tiled<1, 512>(p, smem, grid, a.stream);
    else st = NT == 256 ? launch_tiled<2, 256>(p, smem, grid, a.stream) : launch_tiled<2, 512>(p, smem, grid, a.stream);
    if (want_stats && st == WMH_OK) {
        unsigned long long h[7] = {0};
        cudaMemcpyAsync(h, ctr, sizeof h, cudaMemcpyDeviceToHost, a.stream);
        cudaStreamSynchronize(a.stream);
        const unsigned long long tiles = h[1] + h[2] + h[3] + h[4];
        fprintf(stderr, "[wmh tiled] R=%d SW=%d NT=%d grid=%d items=%lld hchunk=%d tiles C4=%llu C8=%llu C16=%llu C32=%llu mean_s=%.5f\n",
                R, SW, NT, grid, (long long)p.n_items, hchunk, h[1], h[2], h[3], h[4],
                tiles ? (double)h[6] / 1e9 / (double)tiles : 0.0);
    }
    cudaFreeAsync(scratch, a.stream);
    return st;
}

}  // namespace wmh
