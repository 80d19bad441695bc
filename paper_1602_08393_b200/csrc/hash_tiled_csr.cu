// hash_tiled_csr.cu -- WMH_ALGO_TILED for CSR rows (sparse, large D).
//
// Same idea as the dense tiled kernel -- each draw r_t of hash j is shared by
// a tile of rows (the stream does not depend on x) -- but a sparse
// row cannot be expanded in shared memory, so a tile is described by:
//   * an open-addressed table of its nonzeros keyed by column
//     (slot = col << 24 | local row << 8 | x), duplicates allowed;
//   * a bitmap over cell buckets (bucket = r >> S) marking every bucket that
//     touches a green cell [CompToM[c], CompToM[c] + x) of any tile row --
//     a conservative filter in front of the exact ISGREEN.
// A warp takes a hash j; lane = draw: each lane draws r_t (a6), drops it if
// its bucket is cold (almost every draw when s is small), else finds
// c = IntToComp[r] and off = r - CompToM[c] (Alg. 5) and probes the
// table: every tile row with x_c > off is green at t, and the first such t
// per row is kept with a shared atomicMin.  The warp walks the stream 32
// draws at a time until every row of the tile has its first green or the
// cap is reached; h = first t + 1, else cap (Alg. 3 / Def.; R9).
#include <stdio.h>
#include <stdlib.h>

#include "common.cuh"

namespace wmh {

constexpr int CSR_NT = 512;
constexpr int CSR_NW = CSR_NT / 32;
constexpr int CSR_RB = 256;                       // max rows per block item (and per sub-tile)
constexpr unsigned long long CSR_EMPTY = ~0ull;

struct CsrParams {
    const int64_t *row_ptr;
    const int32_t *col;
    const uint8_t *val;
    int64_t n_rows;
    int64_t n_blocks;
    int rb;                      // rows per block item
    int n_hchunks, hchunk;
    int64_t n_items;
    uint32_t k, cap, M, uni_m;
    uint64_t S;
    int bshift;                  // bucket = r >> bshift
    int bm_words;                // bitmap words
    int hbits;                   // table slots = 1 << hbits
    int cap_nnz;                 // max nonzeros per sub-tile
    const uint32_t *pack;        // (c << 8) | (r - CompToM[c]) per cell
    const uint32_t *comp_to_m;
    void *sig;
    unsigned long long *n_sat;
    unsigned long long *item_ctr;
};

__device__ __forceinline__ uint32_t col_hash(uint32_t c, int hbits) {
    return (c * 0x9E3779B1u) >> (32 - hbits);
}

template <int SIGB>
__device__ __forceinline__ void csr_store(void *sig, int64_t idx, uint32_t h) {
    if (SIGB == 1) reinterpret_cast<uint8_t *>(sig)[idx] = (uint8_t)h;
    else reinterpret_cast<uint16_t *>(sig)[idx] = (uint16_t)h;
}

__device__ __forceinline__ uint32_t csr_cell(const CsrParams &p, uint32_t r) {
    if (p.uni_m) {
        uint32_t c = r / p.uni_m;
        return (c << 8) | (r - c * p.uni_m);
    }
    return __ldg(p.pack + r);
}

// One row too long for a tile: lanes = hashes, each lane walks its stream and
// looks x_c up by binary search over the row's columns (Sec. 3.3's search,
// P:274).  Rare (rows with more nonzeros than a tile holds).
template <int SIGB>
__device__ void big_row(const CsrParams &p, int64_t n, uint32_t j0, uint32_t j1, unsigned long long &sat) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t a = p.row_ptr[n], b = p.row_ptr[n + 1];
    for (uint32_t j = j0 + warp * 32 + lane; j < j1; j += CSR_NW * 32) {
        const uint64_t keyj = p.S ^ ((uint64_t)j << 32);
        uint32_t h = p.cap;
        bool found = false;
        for (uint32_t t = 0; t < p.cap; t++) {
            const uint32_t cell = csr_cell(p, mulhi_range(splitmix64(keyj ^ t), p.M));
            const uint32_t c = cell >> 8, off = cell & 0xFFu;
            int64_t lo = a, hi = b;
            while (lo < hi) {
                int64_t mid = (lo + hi) >> 1;
                if ((uint32_t)__ldg(p.col + mid) < c) lo = mid + 1;
                else hi = mid;
            }
            if (lo < b && (uint32_t)__ldg(p.col + lo) == c && (uint32_t)__ldg(p.val + lo) > off) {
                h = t + 1;
                found = true;
                break;
            }
        }
        sat += !found;
        csr_store<SIGB>(p.sig, n * (int64_t)p.k + j, h);
    }
}

template <int SIGB, int DPL>   // DPL: draws per lane per loop iteration (independent SplitMix64 chains)
__global__ void __launch_bounds__(CSR_NT, 1) hash_tiled_csr_kernel(const CsrParams p) {
    extern __shared__ __align__(16) unsigned long long csmem[];
    const int H = 1 << p.hbits;
    unsigned long long *slots = csmem;                                         // [H]
    uint32_t *bm = reinterpret_cast<uint32_t *>(slots + H);                    // [bm_words]
    uint32_t *best_all = bm + p.bm_words;                                      // [NW][RB]
    uint32_t *found_all = best_all + CSR_NW * CSR_RB;                          // [NW]
    uint2 *hq_all = reinterpret_cast<uint2 *>(found_all + CSR_NW);             // [NW][128] queued hot draws
    uint16_t *trow = reinterpret_cast<uint16_t *>(hq_all + CSR_NW * 128);      // [RB+1] sub-tile starts
    uint8_t *alive = reinterpret_cast<uint8_t *>(trow + CSR_RB + 2);           // [RB]
    __shared__ long long s_item;
    __shared__ int s_ntiles, s_hash, s_nalive;

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t *best = best_all + warp * CSR_RB;
    volatile uint32_t *found = found_all + warp;
    uint2 *hq = hq_all + warp * 128;
    unsigned long long sat = 0;

    for (;;) {
        __syncthreads();
        if (threadIdx.x == 0) s_item = (long long)atomicAdd(p.item_ctr, 1ull);
        __syncthreads();
        const long long item = s_item;
        if (item >= p.n_items) break;
        const int64_t blk = item / p.n_hchunks;
        const int hc = (int)(item % p.n_hchunks);
        const int64_t r0 = blk * p.rb;
        const int nrb = (int)min((int64_t)p.rb, p.n_rows - r0);
        const uint32_t j0 = (uint32_t)hc * p.hchunk, j1 = min(p.k, j0 + (uint32_t)p.hchunk);

        // ---- cut the block into sub-tiles of <= cap_nnz nonzeros (greedy) -----
        if (threadIdx.x == 0) {
            int nt = 0;
            long long acc = 0;
            trow[0] = 0;
            for (int i = 0; i < nrb; i++) {
                const long long len = p.row_ptr[r0 + i + 1] - p.row_ptr[r0 + i];
                if (i > trow[nt] && acc + len > p.cap_nnz) { trow[++nt] = (uint16_t)i; acc = 0; }
                acc += len;
            }
            trow[++nt] = (uint16_t)nrb;
            s_ntiles = nt;
        }
        __syncthreads();
        const int ntiles = s_ntiles;

        for (int ti = 0; ti < ntiles; ti++) {
            const int a = trow[ti], b = trow[ti + 1];     // local rows [a, b)
            const int64_t ga = r0 + a;
            const int64_t e0 = p.row_ptr[ga], e1 = p.row_ptr[r0 + b];
            if (e1 - e0 > p.cap_nnz) {                     // a single oversized row
                big_row<SIGB>(p, ga, j0, j1, sat);
                __syncthreads();
                continue;
            }
            // ---- a5: build the tile's column table and cell-bucket filter ----
            for (int i = threadIdx.x; i < H; i += CSR_NT) slots[i] = CSR_EMPTY;
            for (int i = threadIdx.x; i < p.bm_words; i += CSR_NT) bm[i] = 0u;
            if (threadIdx.x == 0) { s_hash = 0; s_nalive = 0; }
            __syncthreads();
            for (int r = a + warp; r < b; r += CSR_NW) {
                const int64_t ra = p.row_ptr[r0 + r], rz = p.row_ptr[r0 + r + 1];
                uint32_t any = 0;
                for (int64_t e = ra + lane; e < rz; e += 32) {
                    const uint32_t c = (uint32_t)__ldg(p.col + e), x = __ldg(p.val + e);
                    if (x == 0) continue;
                    any = 1;
                    const unsigned long long key = ((unsigned long long)c << 24) | ((unsigned long long)(r - a) << 8) | x;
                    uint32_t s = col_hash(c, p.hbits);
                    while (atomicCAS(&slots[s], CSR_EMPTY, key) != CSR_EMPTY) s = (s + 1) & (H - 1);
                    const uint32_t start = __ldg(p.comp_to_m + c);
                    const uint32_t b0 = start >> p.bshift, b1 = (start + x - 1) >> p.bshift;
                    for (uint32_t bk = b0; bk <= b1; bk++) atomicOr(&bm[bk >> 5], 1u << (bk & 31));
                }
                any = __any_sync(0xFFFFFFFFu, any);
                if (lane == 0) {
                    alive[r - a] = (uint8_t)any;
                    if (any) atomicAdd(&s_nalive, 1);
                }
            }
            __syncthreads();
            const int nt_rows = b - a, nalive = s_nalive;

            // ---- hashes: one warp per hash, lane = draw ----------------------
            for (;;) {
                int jj = 0;
                if (lane == 0) jj = atomicAdd(&s_hash, 1);
                const uint32_t j = j0 + (uint32_t)__shfl_sync(0xFFFFFFFFu, jj, 0);
                if (j >= j1) break;
                for (int i = lane; i < nt_rows; i += 32) best[i] = 0xFFFFFFFFu;
                if (lane == 0) *found = 0;
                __syncwarp();
                const uint64_t keyj = p.S ^ ((uint64_t)j << 32);
                // Draws that pass the bucket filter are queued (per warp) and
                // resolved 32 at a time, so the exact check -- an L2 lookup of
                // the packed cell and a table probe -- runs with every lane busy.
                // The first green per row is a min over t, so order is free.
                auto resolve = [&](int count) {
                    if (lane < count) {
                        const uint2 q = hq[lane];                     // (r, t)
                        const uint32_t cell = csr_cell(p, q.x);
                        const uint32_t c = cell >> 8, off = cell & 0xFFu;
                        for (uint32_t s = col_hash(c, p.hbits);; s = (s + 1) & (H - 1)) {
                            const unsigned long long e = slots[s];
                            if (e == CSR_EMPTY) break;
                            if ((uint32_t)(e >> 24) == c && (uint32_t)(e & 0xFFu) > off) {
                                const uint32_t row = (uint32_t)(e >> 8) & 0xFFFFu;
                                if (atomicMin(&best[row], q.y) == 0xFFFFFFFFu) atomicAdd((uint32_t *)found, 1u);
                            }
                        }
                    }
                    __syncwarp();
                    const uint2 k1 = hq[lane + 32], k2 = hq[lane + 64], k3 = hq[lane + 96];   // keep the overflow
                    __syncwarp();
                    hq[lane] = k1;
                    hq[lane + 32] = k2;
                    hq[lane + 64] = k3;
                    __syncwarp();
                };
                int qn = 0;
                const unsigned lt = (1u << lane) - 1;
                // two independent draws per lane per iteration (t0 + lane, t0 + 32 + lane)
                // give the scheduler two SplitMix64 chains to interleave
                for (uint32_t t0 = 0; t0 < p.cap && (int)*found < nalive; t0 += 32 * DPL) {
                    uint32_t rr[DPL];
                    bool hot[DPL];
#pragma unroll
                    for (int u = 0; u < DPL; u++) {
                        const uint32_t t = t0 + 32 * u + lane;
                        rr[u] = mulhi_range(splitmix64(keyj ^ (uint64_t)t), p.M);
                        const uint32_t bk = rr[u] >> p.bshift;
                        hot[u] = t < p.cap && ((bm[bk >> 5] >> (bk & 31)) & 1u);
                    }
#pragma unroll
                    for (int u = 0; u < DPL; u++) {
                        const unsigned hm = __ballot_sync(0xFFFFFFFFu, hot[u]);
                        if (hot[u]) hq[qn + __popc(hm & lt)] = make_uint2(rr[u], t0 + 32 * u + lane);
                        qn += __popc(hm);
                    }
                    __syncwarp();
                    while (qn >= 32) { resolve(32); qn -= 32; }
                }
                if (qn > 0) resolve(qn);                              // flush (the loop may end early)
                // ---- a9: first green t + 1, or the cap ----------------------------
                for (int i = lane; i < nt_rows; i += 32) {
                    const uint32_t bt = best[i];
                    const bool sat_i = bt == 0xFFFFFFFFu;
                    csr_store<SIGB>(p.sig, (r0 + a + i) * (int64_t)p.k + j, sat_i ? p.cap : bt + 1);
                    sat += sat_i;
                }
                __syncwarp();
            }
            __syncthreads();
        }
    }
    if (p.n_sat) {
        for (int o = 16; o; o >>= 1) sat += __shfl_xor_sync(0xFFFFFFFFu, sat, o);
        if (lane == 0 && sat) atomicAdd(p.n_sat, sat);
    }
}

wmh_status launch_hash_tiled_csr(const HashArgs &a, bool *handled) {
    *handled = false;
    int dev = 0;
    cudaGetDevice(&dev);
    int smem_optin = 0;
    cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    const uint32_t M = (uint32_t)a.L->M;
    // cell-bucket filter: <= 2^19 bits (64 KB)
    int bshift = 0;
    while (((uint64_t)M + (1ull << bshift) - 1) >> bshift > (1ull << 19)) bshift++;
    // bitmap words rounded to 16 B so the arrays after it stay 8/16-byte aligned
    const int bm_words = (((int)((((uint64_t)M + (1ull << bshift) - 1) >> bshift) + 31) / 32) + 3) & ~3;
    const size_t fixed = (size_t)bm_words * 4 + (size_t)CSR_NW * CSR_RB * 4 + CSR_NW * 4 + (size_t)CSR_NW * 128 * 8 +
                         (CSR_RB + 2) * 2 + CSR_RB + 64;
    if ((size_t)smem_optin < fixed + 8 * 1024) return WMH_OK;
    int hbits = 0;
    while (((size_t)8 << (hbits + 1)) + fixed <= (size_t)smem_optin) hbits++;
    if (hbits < 10) return WMH_OK;
    const int H = 1 << hbits;
    const size_t smem = fixed + (size_t)8 * H;
    *handled = true;

    CsrParams p;
    p.row_ptr = a.rows.row_ptr;
    p.col = a.rows.col;
    p.val = a.rows.val;
    p.n_rows = a.rows.n_rows;
    const double avg = a.rows.n_rows ? (double)a.rows.nnz / (double)a.rows.n_rows : 1.0;
    p.cap_nnz = (int)(H * 0.6);
    int rb = (int)min(256.0, max(32.0, 8.0 * p.cap_nnz / max(avg, 1.0)));
    rb = (rb + 31) / 32 * 32;
    p.rb = min(rb, CSR_RB);
    p.n_blocks = (a.rows.n_rows + p.rb - 1) / p.rb;
    const int sms = num_sms();
    // hash chunks: enough items to balance the SMs, but >= 4 hashes per warp so
    // the warps of a CTA stay busy between the per-sub-tile barriers
    int n_hchunks = (int)max((int64_t)1, min((int64_t)a.k / (4 * CSR_NW), ((int64_t)sms * 6 + p.n_blocks - 1) / p.n_blocks));
    const int hchunk = (int)((a.k + n_hchunks - 1) / n_hchunks);
    n_hchunks = (int)((a.k + hchunk - 1) / hchunk);
    p.n_hchunks = n_hchunks;
    p.hchunk = hchunk;
    p.n_items = p.n_blocks * n_hchunks;
    p.k = a.k;
    p.cap = a.cap;
    p.M = M;
    p.uni_m = (a.L->flags & WMH_LAYOUT_UNIFORM) ? a.L->uniform_m : 0u;
    p.S = a.S;
    p.bshift = bshift;
    p.bm_words = bm_words;
    p.hbits = hbits;
    p.pack = a.L->cell_pack;
    p.comp_to_m = a.L->comp_to_m;
    p.sig = a.sig;
    p.n_sat = a.n_sat;

    unsigned long long *ctr = nullptr;
    WMH_CUDA_TRY(cudaMallocAsync((void **)&ctr, sizeof(unsigned long long), a.stream), "csr scratch alloc");
    WMH_CUDA_TRY(cudaMemsetAsync(ctr, 0, sizeof(unsigned long long), a.stream), "csr counter memset");
    p.item_ctr = ctr;
    const int grid = (int)min((int64_t)sms, p.n_items);
    // independent SplitMix64 chains per lane: 4 measured best on c3 (119 vs 126 vs 141 ms for 4 / 2 / 1)
    static const int dpl = getenv("WMH_CSR_DPL") ? atoi(getenv("WMH_CSR_DPL")) : 4;
    auto go = [&](auto kern) -> wmh_status {
        WMH_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem), "csr smem attr");
        kernel_timer_begin(a.stream);
        kern<<<grid, CSR_NT, smem, a.stream>>>(p);
        kernel_timer_end(a.stream);
        return WMH_OK;
    };
    wmh_status lst;
    if (a.sig_bytes == 1)
        lst = dpl == 1 ? go(hash_tiled_csr_kernel<1, 1>) : dpl == 4 ? go(hash_tiled_csr_kernel<1, 4>) : go(hash_tiled_csr_kernel<1, 2>);
    else
        lst = dpl == 1 ? go(hash_tiled_csr_kernel<2, 1>) : dpl == 4 ? go(hash_tiled_csr_kernel<2, 4>) : go(hash_tiled_csr_kernel<2, 2>);
    if (lst != WMH_OK) { cudaFreeAsync(ctr, a.stream); return lst; }
    WMH_LAUNCH_CHECK("hash_tiled_csr launch");
    if (getenv("WMH_TILED_STATS"))
        fprintf(stderr, "[wmh tiled csr] H=%d cap_nnz=%d rb=%d blocks=%lld hchunk=%d bshift=%d bm_words=%d smem=%zu\n", H,
                p.cap_nnz, p.rb, (long long)p.n_blocks, hchunk, bshift, bm_words, smem);
    cudaFreeAsync(ctr, a.stream);
    return WMH_OK;
}

}  // namespace wmh
