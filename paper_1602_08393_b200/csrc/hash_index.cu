// hash_index.cu -- WMH_ALGO_INDEX: the draw stream, filed by cell.
//
// The draws r_{j,t} of hash j do not depend on the vector: the paper requires
// the same random sequence for every vector, and Theorem 1's proof
// rests on exactly that.  So instead of drawing until green for
// every (row, j) -- Alg. 3, expected 1/s draws per hash (Theorem 2)
// -- a call draws every (j, t < T) ONCE and files it under its cell r_{j,t}.
// The green cells of a row x are the intervals [CompToM[c], CompToM[c] + x_c)
// of its nonzero coordinates (Eq. 4; reading R2), so
//
//     h_j(x) = 1 + min { t < T_x : (j, t) filed under a green cell of x }
//
// is Alg. 3's first green draw, found by visiting only the row's green draws
// (k * T_x * s of them in expectation, s = |x|_1 / M, Eq. 17) instead of
// testing k / s draws.  A hash with no green draw below T_x continues with
// Alg. 3's own loop from t = T_x (draw-parallel: lane = draw, ballot, first
// set lane) up to the cap (reading R9).  Both parts compute min{t : r_t green}
// -- bit-identical to the oracle by construction, for any T_x.
//
// The per-call index (device scratch), NESTED epochs:
//   epoch e holds every draw t < B[e+1];  B = 32, 64, ..., 512 (x2), 2048, ... (x4), T
//   key     = e * M + r                    (epoch-major, then cell)
//   pos     uint32[E*M + 1]: epoch e's entries of cells [lo, hi) are
//           vals[pos[e*M + lo] .. pos[e*M + hi])
//   vals    uint32: (j << 16) | t          (k <= 65536, t < cap <= 65535)
// A row picks ONE epoch e_x from its own s before visiting (T_x = B[e_x + 1]):
// the one minimising the expected entries k*T*s plus the expected fallback
// draws k*(1-s)^T*min(1/s, cap - T) (reading R17: a scheduling choice; the
// result does not depend on it), then reads one range per nonzero coordinate.
//
// Build, without global atomics (a two-pass partition + per-chunk counting
// sort): keys are cut into chunks of 2^cb consecutive keys;
//   A  each CTA counts its slice of the draws per chunk (shared histogram)
//   -  exclusive scan of the (chunk, CTA) counts, chunk-major
//   B  each CTA re-draws its slice and writes (local key, val) pairs to its
//      private cursor inside each chunk's bucket
//   C  one CTA per chunk: counting sort of its bucket by local key in shared
//      memory; writes pos[] of the chunk's keys and the sorted vals.
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>
#include <type_traits>

#include "common.cuh"

namespace wmh {

constexpr uint32_t IX_NONE = 0xFFFFFFFFu;      // no green draw below the row's horizon yet
constexpr uint32_t IX_SAT = 0xFFFFFFFEu;       // no green draw below the cap
constexpr unsigned FULL = 0xFFFFFFFFu;
constexpr int IX_U = 8;                        // windows in flight per warp step
constexpr int IX_FB = 4;                       // fallback hashes per warp at once

// first epoch that holds draw t (it is also in every later one)
__device__ __forceinline__ int ix_first_epoch(uint32_t t, const IxEpochs &ep) {
    int e = 0;
#pragma unroll
    for (int i = 1; i < IX_MAXE; i++)
        if (i < ep.E && t >= ep.B[i]) e = i;
    return e;
}

// ------------------------------------------------------------------ build
struct IxBuild {
    uint64_t S;
    uint32_t k, T, M;
    IxEpochs ep;
    int cb[IX_MAXE];             // epoch e is cut into chunks of 2^cb[e] consecutive cells
    uint32_t cbase[IX_MAXE + 1]; // first chunk of epoch e; cbase[E] = n_chunks
    int cb_max;
    uint32_t n_chunks;
    uint64_t n_keys;             // E * M
    uint64_t n_draws;            // k * T
    uint64_t per_cta;            // draws per CTA slice (passes A and B)
    int n_cta;
};

template <bool WRITE>
__global__ void __launch_bounds__(512) ix_partition(const IxBuild b, uint32_t *__restrict__ H,
                                                    uint32_t *__restrict__ tmp) {
    extern __shared__ uint32_t cnt[];          // [n_chunks]: counts (A) or cursors (B)
    for (uint32_t i = threadIdx.x; i < b.n_chunks; i += blockDim.x)
        cnt[i] = WRITE ? H[(uint64_t)i * b.n_cta + blockIdx.x] : 0u;
    __syncthreads();
    const uint64_t d0 = (uint64_t)blockIdx.x * b.per_cta;
    const uint64_t d1 = min(b.n_draws, d0 + b.per_cta);
    for (uint64_t d = d0 + threadIdx.x; d < d1; d += blockDim.x) {
        const uint32_t j = (uint32_t)(d / b.T), t = (uint32_t)(d - (uint64_t)j * b.T);
        const uint32_t r = mulhi_range(splitmix64(b.S ^ ((uint64_t)j << 32) ^ (uint64_t)t), b.M);
        for (int e = ix_first_epoch(t, b.ep); e < b.ep.E; e++) {
            const uint32_t c = b.cbase[e] + (r >> b.cb[e]);
            if (WRITE) tmp[atomicAdd(cnt + c, 1u)] = (j << 16) | t;   // the cell is re-drawn in C
            else atomicAdd(cnt + c, 1u);
        }
    }
    if (!WRITE) {
        __syncthreads();
        for (uint32_t i = threadIdx.x; i < b.n_chunks; i += blockDim.x)
            H[1 + (uint64_t)i * b.n_cta + blockIdx.x] = cnt[i];
    }
}

constexpr int SC_T = 1024, SC_V = 8, SC_TILE = SC_T * SC_V;

// block-wide exclusive scan (SC_T threads); *total (optional) gets the sum
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t v, uint32_t *total) {
    __shared__ uint32_t ws[SC_T / 32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t u = __shfl_up_sync(FULL, incl, o);
        if (lane >= o) incl += u;
    }
    if (lane == 31) ws[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        const uint32_t w = lane < (int)(blockDim.x >> 5) ? ws[lane] : 0u;
        uint32_t wi = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t u = __shfl_up_sync(FULL, wi, o);
            if (lane >= o) wi += u;
        }
        ws[lane] = wi - w;
        if (total && lane == 31) *total = wi;
    }
    __syncthreads();
    const uint32_t r = ws[warp] + incl - v;
    __syncthreads();
    return r;
}

// C: one CTA (SC_T threads) per chunk: counting sort of the chunk's entries by
// cell (each entry's cell re-drawn from its (j, t)), pos[] of the chunk's cells,
// entries scattered into their sorted slots.
__global__ void __launch_bounds__(SC_T) ix_chunk_sort(const IxBuild b, const uint32_t *__restrict__ H,
                                                      const uint32_t *__restrict__ tmp, uint32_t *__restrict__ pos,
                                                      uint32_t *__restrict__ vals) {
    extern __shared__ uint32_t cnt[];          // [2^cb[e]]
    const uint32_t c = blockIdx.x;
    int e = 0;
    for (int i = 1; i < b.ep.E; i++)
        if (c >= b.cbase[i]) e = i;
    const int cb = b.cb[e];
    const uint32_t r0 = (c - b.cbase[e]) << cb;
    const uint32_t nloc = min(1u << cb, b.M - r0);
    const uint32_t beg = H[(uint64_t)c * b.n_cta];
    const uint32_t end = H[(uint64_t)(c + 1) * b.n_cta];
    for (uint32_t i = threadIdx.x; i < nloc; i += SC_T) cnt[i] = 0;
    __syncthreads();
    for (uint32_t p = beg + threadIdx.x; p < end; p += SC_T) {
        const uint32_t v = tmp[p];
        const uint32_t r = mulhi_range(splitmix64(b.S ^ ((uint64_t)(v >> 16) << 32) ^ (uint64_t)(v & 0xFFFFu)), b.M);
        atomicAdd(cnt + (r - r0), 1u);
    }
    __syncthreads();
    // exclusive scan of cnt[0..nloc): each thread owns consecutive counters
    const uint32_t per = (nloc + SC_T - 1) / SC_T, i0 = threadIdx.x * per;
    uint32_t s = 0;
    for (uint32_t i = i0; i < min(nloc, i0 + per); i++) s += cnt[i];
    uint32_t run = beg + block_excl_scan(s, nullptr);
    const uint64_t key0 = (uint64_t)e * b.M + r0;
    for (uint32_t i = i0; i < min(nloc, i0 + per); i++) {
        const uint32_t v = cnt[i];
        cnt[i] = run;
        pos[key0 + i] = run;
        run += v;
    }
    if (c + 1 == b.n_chunks && threadIdx.x == 0) pos[b.n_keys] = end;
    __syncthreads();
    for (uint32_t p = beg + threadIdx.x; p < end; p += SC_T) {
        const uint32_t v = tmp[p];
        const uint32_t r = mulhi_range(splitmix64(b.S ^ ((uint64_t)(v >> 16) << 32) ^ (uint64_t)(v & 0xFFFFu)), b.M);
        vals[atomicAdd(cnt + (r - r0), 1u)] = v;
    }
}

// colstart[e * (D + 1) + c] = pos[e * M + CompToM[c]]: the first filed draw of
// column c in epoch e, so a row reads one of its two range bounds from a
// D-sized (L2-resident) array instead of the E*M-sized pos.
__global__ void ix_colstart_kernel(const uint32_t *__restrict__ pos, const uint32_t *__restrict__ c2m, uint32_t uni_m,
                                   int E, uint32_t M, int64_t D, uint32_t *__restrict__ colstart) {
    const int64_t total = (int64_t)E * (D + 1);
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t e = i / (D + 1), c = i - e * (D + 1);
        const uint32_t lo = uni_m ? (uint32_t)c * uni_m : __ldg(c2m + c);
        colstart[i] = pos[(uint64_t)e * M + lo];
    }
}

// In-place inclusive scan of uint32 a[0..n): tile sums, a one-block scan of
// the sums, per-tile scans with the carried offset.
__global__ void __launch_bounds__(SC_T) scan_tile_sums(const uint32_t *__restrict__ a, int64_t n,
                                                       uint32_t *__restrict__ sums) {
    const int64_t base = (int64_t)blockIdx.x * SC_TILE + (int64_t)threadIdx.x * SC_V;
    uint32_t s = 0;
#pragma unroll
    for (int i = 0; i < SC_V; i++)
        if (base + i < n) s += a[base + i];
    __shared__ uint32_t tot;
    block_excl_scan(s, &tot);
    if (threadIdx.x == 0) sums[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(SC_T) scan_sums_excl(uint32_t *__restrict__ sums, int64_t nt) {
    __shared__ uint32_t carry_s;
    uint32_t carry = 0;
    for (int64_t b0 = 0; b0 < nt; b0 += SC_T) {
        const int64_t i = b0 + threadIdx.x;
        const uint32_t v = i < nt ? sums[i] : 0u;
        const uint32_t ex = block_excl_scan(v, &carry_s);
        if (i < nt) sums[i] = carry + ex;
        carry += carry_s;
        __syncthreads();
    }
}

__global__ void __launch_bounds__(SC_T) scan_tile_apply(uint32_t *__restrict__ a, int64_t n,
                                                        const uint32_t *__restrict__ sums) {
    const int64_t base = (int64_t)blockIdx.x * SC_TILE + (int64_t)threadIdx.x * SC_V;
    uint32_t v[SC_V], s = 0;
#pragma unroll
    for (int i = 0; i < SC_V; i++) {
        v[i] = base + i < n ? a[base + i] : 0u;
        s += v[i];
    }
    uint32_t run = sums[blockIdx.x] + block_excl_scan(s, nullptr);
#pragma unroll
    for (int i = 0; i < SC_V; i++) {
        run += v[i];
        if (base + i < n) a[base + i] = run;
    }
}

wmh_status scan_u32_inplace(uint32_t *a, int64_t n, uint32_t *sums, cudaStream_t s) {
    const int64_t nt = (n + SC_TILE - 1) / SC_TILE;
    if (nt == 0) return WMH_OK;
    scan_tile_sums<<<(unsigned)nt, SC_T, 0, s>>>(a, n, sums);
    WMH_LAUNCH_CHECK("index scan sums");
    scan_sums_excl<<<1, SC_T, 0, s>>>(sums, nt);
    WMH_LAUNCH_CHECK("index scan of sums");
    scan_tile_apply<<<(unsigned)nt, SC_T, 0, s>>>(a, n, sums);
    WMH_LAUNCH_CHECK("index scan apply");
    return WMH_OK;
}

// ------------------------------------------------------------- the rows
struct IxParams {
    const void *x;               // dense rows (n_rows x D, uint8 or uint16 weights) or null
    const int64_t *row_ptr;      // CSR
    const int32_t *col;
    const void *val;             // CSR weights (uint8 or uint16)
    int64_t n_rows, D;
    const uint32_t *comp_to_m, *pack, *i2c;   // pack = null for wide layouts
    uint32_t uni_m, M;
    const uint32_t *pos, *vals;
    const uint32_t *colstart;    // [E][D + 1]: pos[e*M + CompToM[c]]
    const uint2 *table;          // (c, r - CompToM[c]) of draws t < T0 of every hash
    IxEpochs ep;
    uint64_t S;
    uint32_t k, cap;
    int capn;                    // CSR rows with nnz <= capn stage their columns in shared memory
    float cf_dense, cf_smem, cf_global;   // cost of one fallback draw / one index entry
    float cf_bitmap;             // ... with the row's column bitmap in shared memory (8 warps)
    int bm_words;                // 8 warps, unstaged CSR rows: ceil(D / 32) when the bitmap fits, else 0
    void *sig;
    unsigned long long *n_sat;
    unsigned long long *row_ctr;
    const uint32_t *perm;        // rows in processing order (deepest epoch first), or null
    uint8_t *plan;               // optional [n_rows]: the row's plan code (wmh_hash_opts.plan_out)
};

// x_c of the current row: dense byte, or a lower_bound over the CSR slice
// (its columns staged in shared memory when the row is short enough).
// x_c of the row: dense -> direct; CSR -> with the row's column bitmap bm[]
// (bit c set iff c is a column of the row) and pre[w] = the index of the first
// column in bitmap word w, one shared load plus, for a column of the row, its
// rank; else binary search of c among the row's columns, in shared memory when
// staged (scol), else first over the staged sample samp[i] = col[i * sd] (ns
// entries) and then among the <= sd - 1 columns of one block in global memory
// (one or two cache lines)
template <bool CSR, typename W>
__device__ __forceinline__ uint32_t ix_row_x(const IxParams &p, const W *xrow, const uint32_t *scol,
                                             int64_t e0, int n, uint32_t c, const uint32_t *samp = nullptr,
                                             int ns = 0, int sd = 1, const uint32_t *bm = nullptr,
                                             const uint16_t *pre = nullptr) {
    const W *val = reinterpret_cast<const W *>(p.val);
    if (!CSR) return scol ? (uint32_t)reinterpret_cast<const W *>(scol)[c] : (uint32_t)__ldg(xrow + c);
    if (bm) {                                    // the row's column bitmap: one shared load decides
        const uint32_t w = bm[c >> 5], b = c & 31u;    // x_c = 0 (most draws); else the rank of c
        if (!((w >> b) & 1u)) return 0u;               // among the row's columns gives its weight
        const uint32_t rk = pre[c >> 5] + __popc(w & ((1u << b) - 1u));
        WMH_DASSERT(rk < (uint32_t)n && (uint32_t)__ldg(p.col + e0 + rk) == c);
        return (uint32_t)__ldg(val + e0 + rk);
    }
    int lo = 0, hi = n;
    if (!scol && samp) {
        int a = 0, b = ns;                       // first i with samp[i] >= c
        while (a < b) {
            const int mid = (a + b) >> 1;
            if (samp[mid] < c) a = mid + 1;
            else b = mid;
        }
        if (a < ns && samp[a] == c) return (uint32_t)__ldg(val + e0 + (int64_t)a * sd);
        if (a == 0) return 0u;
        lo = (a - 1) * sd + 1;                   // col[(a-1) * sd] < c < col[a * sd]
        hi = min(n, a * sd);
    }
    if (scol) {
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (scol[mid] < c) lo = mid + 1;
            else hi = mid;
        }
        return (lo < n && scol[lo] == c) ? (uint32_t)__ldg(val + e0 + lo) : 0u;
    }
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if ((uint32_t)__ldg(p.col + e0 + mid) < c) lo = mid + 1;
        else hi = mid;
    }
    return (lo < n && (uint32_t)__ldg(p.col + e0 + lo) == c) ? (uint32_t)__ldg(val + e0 + lo) : 0u;
}

template <int NW>
__device__ __forceinline__ unsigned long long block_sum(unsigned long long a) {
    __shared__ unsigned long long ra[NW];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o; o >>= 1) a += __shfl_xor_sync(FULL, a, o);
    if (lane == 0) ra[warp] = a;
    __syncthreads();
    a = 0;
#pragma unroll
    for (int w = 0; w < NW; w++) a += ra[w];
    __syncthreads();
    return a;
}

// The row's epoch: minimise k*T*s (entries) + k*(1-s)^T * per-hash fallback draws * cf.
__device__ __forceinline__ int ix_plan(const IxParams &p, float s, float cf) {
    if (s >= 1.f) return 0;
    const float l2 = log2f(1.f - s);
    int best_e = 0;
    float best = INFINITY;
    for (int e = 0; e < p.ep.E; e++) {
        const float T = (float)p.ep.B[e + 1];
        const float rest = T >= (float)p.cap ? 0.f : fmaxf(32.f, fminf(1.f / s, (float)p.cap - T));
        const float cost = (float)p.k * (T * s + exp2f(T * l2) * rest * cf);
        if (cost < best) { best = cost; best_e = e; }
    }
    return best_e;
}

// Processing order: rows grouped by the epoch their plan picks, deepest first,
// so the CTAs resident at any time read the same epoch's pos[] / vals[] (one
// epoch's tables fit L2 where all of them do not) and the heaviest rows start
// first.  The order changes nothing but the schedule.
template <bool CSR, typename W>
__global__ void __launch_bounds__(256) ix_order_count(const IxParams p, uint8_t *__restrict__ row_epoch,
                                                      unsigned int *__restrict__ cnt) {
    const int lane = threadIdx.x & 31;
    const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t r = w0; r < p.n_rows; r += nw) {
        unsigned long long xs = 0;
        if (CSR) {
            const int64_t a = p.row_ptr[r], b = p.row_ptr[r + 1];
            for (int64_t i = a + lane; i < b; i += 32) xs += __ldg(reinterpret_cast<const W *>(p.val) + i);
        } else {
            const W *x = reinterpret_cast<const W *>(p.x) + r * p.D;
            for (int64_t i = lane; i < p.D; i += 32) xs += __ldg(x + i);
        }
        for (int o = 16; o; o >>= 1) xs += __shfl_xor_sync(0xFFFFFFFFu, xs, o);
        const int e = xs ? ix_plan(p, (float)((double)xs / (double)p.M), CSR ? (p.bm_words ? p.cf_bitmap : p.cf_global) : p.cf_dense) : 0;
        if (lane == 0) {
            row_epoch[r] = (uint8_t)e;
            atomicAdd(cnt + e, 1u);
        }
    }
}

__global__ void __launch_bounds__(256) ix_order_scatter(int64_t n_rows, int E, const uint8_t *__restrict__ row_epoch,
                                                        const unsigned int *__restrict__ cnt,
                                                        unsigned int *__restrict__ cursor, uint32_t *__restrict__ perm) {
    __shared__ unsigned int base[IX_MAXE];
    if (threadIdx.x == 0) {                      // deepest epoch first
        unsigned int run = 0;
        for (int e = E - 1; e >= 0; e--) {
            base[e] = run;
            run += cnt[e];
        }
    }
    __syncthreads();
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n_rows; r += (int64_t)gridDim.x * blockDim.x) {
        const int e = row_epoch[r];
        const unsigned peers = __match_any_sync(__activemask(), e);
        const int leader = __ffs(peers) - 1, lane = threadIdx.x & 31;
        unsigned int b0 = 0;
        if (lane == leader) b0 = atomicAdd(cursor + e, (unsigned)__popc(peers));
        b0 = __shfl_sync(peers, b0, leader);
        perm[base[e] + b0 + __popc(peers & ((1u << lane) - 1))] = (uint32_t)r;
    }
}

// Block-wide exclusive scan of a 64-bit value (NW warps); *total gets the sum.
template <int NW>
__device__ __forceinline__ unsigned long long block_excl_scan64(unsigned long long v, unsigned long long *total) {
    __shared__ unsigned long long ws[NW];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned long long incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long u = __shfl_up_sync(FULL, incl, o);
        if (lane >= o) incl += u;
    }
    if (lane == 31) ws[warp] = incl;
    __syncthreads();
    unsigned long long before = 0, all = 0;
#pragma unroll
    for (int w = 0; w < NW; w++) {
        const unsigned long long t = ws[w];
        if (w < warp) before += t;
        all += t;
    }
    __syncthreads();
    *total = all;
    return before + incl - v;
}

// One CTA of NW warps per row (rows claimed from a counter).  Per batch of up
// to NT*8 nonzero coordinates: (1) every thread resolves the ranges of its 8
// coordinates (all pos[] loads in flight together) and the non-empty ranges
// are compacted into shared memory with the exclusive prefix of their lengths;
// (2) the warps walk the concatenated entries 32 at a time -- lane f takes
// flat index base + f, its range found from the boundaries that fall inside
// the window (one shared load, one OR-reduction, one popc) -- and fold each
// (j, t) into h[j] = min(h[j], t) with a shared-memory atomic.
// register budget: 64 at 1 and 8 warps, 48 at 2 and 4 (ptxas' own choice
// spilled the 8-warp variant at 48; 40 at 2 warps ran c3 19% slower)
template <int SIGB, bool CSR, int NW, typename W>
__global__ void __maxnreg__((NW == 2 || NW == 4) ? 48 : 64) hash_index_kernel(const IxParams p) {
    const W *pval = reinterpret_cast<const W *>(p.val);
    constexpr int NT = NW * 32, ITEMS = 8, CAPR = NT * ITEMS;
    extern __shared__ uint32_t smem[];
    uint32_t *h = smem;                          // [k] first green t per hash
    uint32_t *ra = h + p.k;                      // [CAPR] range start in vals minus its flat offset (mod 2^32)
    uint32_t *rp = ra + CAPR;                    // [CAPR + 33] exclusive prefix of range lengths, FULL-padded
    uint32_t *scol_buf = rp + CAPR + 33;         // [capn] staged CSR columns
    __shared__ long long s_row;
    __shared__ uint32_t s_nu, s_qhead;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t lanemask_le = lane == 31 ? FULL : ((2u << lane) - 1u);
    unsigned long long sat = 0;
    for (;;) {
        if (threadIdx.x == 0) s_row = (long long)atomicAdd(p.row_ctr, 1ull);
        for (uint32_t j = threadIdx.x; j < p.k; j += NT) h[j] = IX_NONE;
        __syncthreads();
        if (s_row >= p.n_rows) break;
        const long long row = p.perm ? (long long)p.perm[s_row] : s_row;
        int64_t e0 = 0;
        int n;
        const W *xrow = nullptr;
        if (CSR) {
            e0 = p.row_ptr[row];
            n = (int)(p.row_ptr[row + 1] - e0);
        } else {
            xrow = reinterpret_cast<const W *>(p.x) + row * p.D;
            n = (int)p.D;
        }
        constexpr int PER_WORD = 4 / sizeof(W);          // weights per 32-bit word
        const bool staged = CSR ? n <= p.capn : (p.D % PER_WORD) == 0 && (n / PER_WORD) <= p.capn;
        // ---- |x|_1 (and the columns of a short CSR row into shared memory)
        unsigned long long xs = 0;
        if (CSR) {
            for (int i = threadIdx.x; i < n; i += NT) {
                xs += __ldg(pval + e0 + i);
                if (staged) scol_buf[i] = (uint32_t)__ldg(p.col + e0 + i);
            }
        } else if ((p.D % PER_WORD) == 0) {
            const uint32_t *x4 = reinterpret_cast<const uint32_t *>(xrow);
            for (int i = threadIdx.x; i < n / PER_WORD; i += NT) {
                const uint32_t w = __ldg(x4 + i);
                xs += sizeof(W) == 1 ? __dp4a(w, 0x01010101u, 0u) : (w & 0xFFFFu) + (w >> 16);
                if (staged) scol_buf[i] = w;             // the dense row, for the fallback lookups
            }
        } else {
            for (int i = threadIdx.x; i < n; i += NT) xs += __ldg(xrow + i);
        }
        xs = block_sum<NW>(xs);
        // plan code (tests): epoch | staged << 4 | fallback ran << 5 | several range batches << 6 | zero row << 7
        uint32_t plan = (staged ? 16u : 0u) | (n > CAPR ? 64u : 0u);
        if (xs == 0) {                           // an all-zero row never turns green (reading R12)
            for (uint32_t j = threadIdx.x; j < p.k; j += NT) h[j] = IX_SAT;
            plan |= 128u;
        } else {
            const float s = (float)((double)xs / (double)p.M);
            const int e = ix_plan(p, s, CSR ? (staged ? p.cf_smem : (p.bm_words && n < 65536) ? p.cf_bitmap : p.cf_global) : p.cf_dense);
            plan |= (uint32_t)e;
            const uint32_t T = p.ep.B[e + 1];
            const uint32_t *pe = p.pos + (uint64_t)e * p.M;
            const uint32_t *ce = p.colstart + (uint64_t)e * (p.D + 1);
            for (int b0 = 0; b0 < n; b0 += CAPR) {
                // ---- (1) ranges of this thread's 8 coordinates
                const int i0 = b0 + threadIdx.x * ITEMS;
                uint32_t xv[ITEMS], lo[ITEMS];
                if (!CSR && sizeof(W) == 1 && ((p.D & 7) == 0) && i0 + ITEMS <= n) {
                    const uint2 w = __ldg(reinterpret_cast<const uint2 *>(xrow + i0));
#pragma unroll
                    for (int q = 0; q < ITEMS; q++) xv[q] = ((q < 4 ? w.x : w.y) >> (8 * (q & 3))) & 0xFFu;
                } else if (!CSR && sizeof(W) == 2 && ((p.D & 7) == 0) && i0 + ITEMS <= n) {
                    const uint4 w = __ldg(reinterpret_cast<const uint4 *>(xrow + i0));
                    const uint32_t ww[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
                    for (int q = 0; q < ITEMS; q++) xv[q] = (ww[q >> 1] >> (16 * (q & 1))) & 0xFFFFu;
                } else {
#pragma unroll
                    for (int q = 0; q < ITEMS; q++)
                        xv[q] = i0 + q < n ? (CSR ? (uint32_t)__ldg(pval + e0 + i0 + q) : (uint32_t)__ldg(xrow + i0 + q)) : 0u;
                }
#pragma unroll
                for (int q = 0; q < ITEMS; q++) {
                    uint32_t c = (uint32_t)(i0 + q);
                    if (CSR && xv[q]) c = staged ? scol_buf[i0 + q] : (uint32_t)__ldg(p.col + e0 + i0 + q);
                    lo[q] = xv[q] ? (p.uni_m ? c * p.uni_m : __ldg(p.comp_to_m + c)) : 0u;
                }
                uint32_t a[ITEMS], len[ITEMS];
#pragma unroll
                for (int q = 0; q < ITEMS; q++) {
                    // uniform bounds: the column start from the small colstart table
                    // (c = lo / m), else pos at the cell itself
                    a[q] = xv[q] ? __ldg(p.uni_m ? ce + lo[q] / p.uni_m : pe + lo[q]) : 0u;
                    len[q] = xv[q] ? __ldg(pe + lo[q] + xv[q]) : 0u;
                }
                uint32_t cnt = 0, sum = 0;
#pragma unroll
                for (int q = 0; q < ITEMS; q++) {
                    len[q] -= a[q];
                    cnt += len[q] != 0;
                    sum += len[q];
                }
                unsigned long long tot;
                const unsigned long long ex = block_excl_scan64<NW>(((unsigned long long)cnt << 32) | sum, &tot);
                uint32_t slot = (uint32_t)(ex >> 32), f = (uint32_t)ex;
#pragma unroll
                for (int q = 0; q < ITEMS; q++)
                    if (len[q]) {
                        WMH_DASSERT(slot < (uint32_t)CAPR);
                        ra[slot] = a[q] - f;
                        rp[slot] = f;
                        slot++;
                        f += len[q];
                    }
                const uint32_t nr = (uint32_t)(tot >> 32), L = (uint32_t)tot;
                if (threadIdx.x < 33) rp[nr + threadIdx.x] = threadIdx.x ? FULL : L;   // end + padding
                __syncthreads();
                // ---- (2) walk the entries, 32 per window, warps on contiguous window blocks
                const uint32_t nwin = (L + 31) >> 5, per = (nwin + NW - 1) / NW;
                const uint32_t w0 = warp * per, w1 = min(nwin, w0 + per);
                if (w0 < w1) {
                    uint32_t base = w0 << 5;
                    uint32_t o = 0, hi = nr;             // owner of base: last o with rp[o] <= base
                    while (hi - o > 1) {
                        const uint32_t mid = (o + hi) >> 1;
                        if (rp[mid] <= base) o = mid;
                        else hi = mid;
                    }
                    // IX_U windows per step: their ranges are found first (shared loads
                    // only), then all IX_U vals loads are issued, then the atomics --
                    // so a lane keeps IX_U global loads in flight
                    const uint32_t lim = min(L, w1 << 5);
                    for (uint32_t w = w0; w < w1; w += IX_U) {
                        uint32_t addr[IX_U];
#pragma unroll
                        for (int u = 0; u < IX_U; u++) {
                            const uint32_t bu = base + 32u * u;
                            const uint32_t d = rp[o + 1 + lane] - bu;     // padded with FULL past nr
                            uint32_t bit;                              // 1 << d, 0 for d >= 32 (PTX shl clamps)
                            asm("shl.b32 %0, 1, %1;" : "=r"(bit) : "r"(d));
                            const uint32_t m = __reduce_or_sync(FULL, bit);   // uniform
                            const uint32_t own = o + __popc(m & lanemask_le);
                            addr[u] = ra[own] + (bu + lane);                   // = start + (flat - flat start)
                            o += __popc(m);                            // the owner of the next window's base
                        }
                        uint32_t v[IX_U];
#pragma unroll
                        for (int u = 0; u < IX_U; u++)
                            v[u] = base + 32u * u + lane < lim ? __ldg(p.vals + addr[u]) : IX_NONE;
#pragma unroll
                        for (int u = 0; u < IX_U; u++)
                            if (v[u] != IX_NONE) {
                                WMH_DASSERT((v[u] >> 16) < p.k);
                                atomicMin(h + (v[u] >> 16), v[u] & 0xFFFFu);
                            }
                        base += 32u * IX_U;
                    }
                }
                __syncthreads();
            }
            if (T < p.cap) {
                // ---- Alg. 3's loop from t = T for the hashes still without a green
                //      draw: their ids are gathered into a shared list (ra[] is free
                //      now); each warp keeps IX_FB of them in flight, lane = draw
                //      (IX_FB independent lookups per lane), refilling from the list
                const uint32_t *scol = staged ? scol_buf : nullptr;
                using list_t = typename std::conditional<NW == 8, uint16_t, uint32_t>::type;   // k < 2^16
                list_t *list = reinterpret_cast<list_t *>(ra);
                // 8 warps (large k: many fallback hashes per row) on an unstaged CSR
                // row: the row's column bitmap (bit c of bm[] set iff x_c > 0) and the
                // index of the first column of each bitmap word in ra[] (free after
                // phase 2), so most lookups are one shared load (x_c = 0) and the rest
                // a rank plus one global load of the weight; when the bitmap does not
                // fit, a sample of the columns in rp[] turns the ~11 dependent global
                // loads of each lookup into shared-memory steps and one or two global
                // ones (c4: 19.9 -> 18.9 ms; with fewer warps the extra code cost more
                // than it saved, c3 10.0 -> 11.0 ms)
                const uint32_t *samp = nullptr, *bm = nullptr;
                const uint16_t *pre = nullptr;
                int ns = 0, sd = 1;
                if constexpr (CSR && NW == 8) {
                    if (!staged && p.bm_words && n < 65536) {
                        const int bmw = p.bm_words;
                        uint32_t *bmw_s = ra;
                        uint16_t *pre_s = reinterpret_cast<uint16_t *>(ra + bmw);
                        for (int i = threadIdx.x; i < bmw; i += NT) bmw_s[i] = 0u;
                        __syncthreads();
                        for (int i = threadIdx.x; i < n; i += NT) {
                            const uint32_t c = (uint32_t)__ldg(p.col + e0 + i);
                            WMH_DASSERT((c >> 5) < (uint32_t)bmw);
                            atomicOr(bmw_s + (c >> 5), 1u << (c & 31u));
                            // columns strictly ascending: the first of its word sets pre[]
                            if (i == 0 || ((uint32_t)__ldg(p.col + e0 + i - 1) >> 5) != (c >> 5)) pre_s[c >> 5] = (uint16_t)i;
                        }
                        bm = bmw_s;
                        pre = pre_s;
                        list = reinterpret_cast<list_t *>(ra + bmw + ((bmw + 1) >> 1));
                    } else if (!staged) {
                        sd = (n + CAPR - 1) / CAPR;
                        ns = (n + sd - 1) / sd;
                        for (int i = threadIdx.x; i < ns; i += NT) rp[i] = (uint32_t)__ldg(p.col + e0 + (int64_t)i * sd);
                        samp = rp;                // visible after the loop's first __syncthreads
                    }
                }
                for (;;) {
                    if (threadIdx.x == 0) { s_nu = 0; s_qhead = 0; }
                    __syncthreads();
                    for (uint32_t jb = warp * 32; jb < p.k; jb += NT) {
                        const uint32_t jl = jb + lane;
                        const bool need = jl < p.k && h[jl] == IX_NONE;
                        const unsigned m = __ballot_sync(FULL, need);
                        uint32_t base = 0;
                        if (lane == 0 && m) base = atomicAdd(&s_nu, (uint32_t)__popc(m));
                        base = __shfl_sync(FULL, base, 0);
                        const uint32_t slot = base + __popc(m & (lanemask_le >> 1));
                        if (need && slot < (uint32_t)CAPR) list[slot] = (list_t)jl;
                    }
                    __syncthreads();
                    const uint32_t U = min(s_nu, (uint32_t)CAPR);
                    if (U == 0) break;
                    plan |= 32u;
                    if constexpr (NW < 8) {
                    // IX_FB slots per warp, each with its own hash and draw position;
                    // a slot whose hash resolves (or reaches the cap) takes the next
                    // hash from the shared queue at once, so no warp idles behind
                    // another's geometric tail
                    uint32_t jq[IX_FB], tq[IX_FB];
                    unsigned live = 0;
                    {
                        uint32_t q0 = 0;
                        if (lane == 0) q0 = atomicAdd(&s_qhead, (uint32_t)IX_FB);
                        q0 = __shfl_sync(FULL, q0, 0);
#pragma unroll
                        for (int q = 0; q < IX_FB; q++) {
                            jq[q] = q0 + q < U ? list[q0 + q] : 0u;
                            tq[q] = T;
                            if (q0 + q < U) live |= 1u << q;
                        }
                    }
                    while (live) {
                        uint32_t c[IX_FB], off[IX_FB];
#pragma unroll
                        for (int q = 0; q < IX_FB; q++) {
                            c[q] = 0;
                            off[q] = 0xFFFFFFFFu;
                            const uint32_t t = tq[q] + lane;
                            if ((live >> q) & 1u) {
                                if (t < (uint32_t)T0) {                // the call's table of the first draws
                                    const uint2 d = __ldg(p.table + (uint64_t)jq[q] * T0 + t);
                                    c[q] = d.x;
                                    off[q] = d.y;
                                } else if (t < p.cap) {
                                    const uint2 cell = cell_lookup(
                                        mulhi_range(splitmix64(p.S ^ ((uint64_t)jq[q] << 32) ^ (uint64_t)t), p.M),
                                        p.pack, p.uni_m, p.i2c, p.comp_to_m);
                                    c[q] = cell.x;
                                    off[q] = cell.y;
                                }
                            }
                        }
#pragma unroll
                        for (int q = 0; q < IX_FB; q++) {
                            if (!((live >> q) & 1u)) continue;
                            const bool g = off[q] != 0xFFFFFFFFu && off[q] < ix_row_x<CSR, W>(p, xrow, scol, e0, n, c[q], samp, ns, sd, bm, pre);
                            const unsigned gm = __ballot_sync(FULL, g);
                            bool done = false;
                            if (gm) {
                                if (lane == 0) h[jq[q]] = tq[q] + __ffs(gm) - 1;
                                done = true;
                            } else {
                                tq[q] += 32;
                                if (tq[q] >= p.cap) {                  // no green draw before the cap
                                    if (lane == 0) h[jq[q]] = IX_SAT;
                                    done = true;
                                }
                            }
                            if (done) {                                // refill the slot
                                uint32_t nx = 0;
                                if (lane == 0) nx = atomicAdd(&s_qhead, 1u);
                                nx = __shfl_sync(FULL, nx, 0);
                                if (nx < U) {
                                    jq[q] = list[nx];
                                    tq[q] = T;
                                } else {
                                    live &= ~(1u << q);
                                }
                            }
                        }
                    }
                    } else {
                    // 8 warps: static batches of IX_FB hashes (measured: c4 20.3 vs 21.0 ms with the refill)
                    for (uint32_t ub = warp * IX_FB; ub < U; ub += NT / 32 * IX_FB) {
                        uint32_t jq[IX_FB];
                        unsigned live = 0;
#pragma unroll
                        for (int q = 0; q < IX_FB; q++) {
                            jq[q] = ub + q < U ? list[ub + q] : 0u;
                            if (ub + q < U) live |= 1u << q;
                        }
                        uint32_t t0 = T;
                        for (; live && t0 < p.cap; t0 += 32) {
                            const uint32_t t = t0 + lane;
                            uint32_t c[IX_FB], off[IX_FB];
#pragma unroll
                            for (int q = 0; q < IX_FB; q++) {
                                c[q] = 0;
                                off[q] = 0xFFFFFFFFu;
                                if ((live >> q) & 1u) {
                                    if (t < (uint32_t)T0) {            // the call's table of the first draws
                                        const uint2 d = __ldg(p.table + (uint64_t)jq[q] * T0 + t);
                                        c[q] = d.x;
                                        off[q] = d.y;
                                    } else if (t < p.cap) {
                                        const uint2 cell = cell_lookup(
                                            mulhi_range(splitmix64(p.S ^ ((uint64_t)jq[q] << 32) ^ (uint64_t)t), p.M),
                                            p.pack, p.uni_m, p.i2c, p.comp_to_m);
                                        c[q] = cell.x;
                                        off[q] = cell.y;
                                    }
                                }
                            }
#pragma unroll
                            for (int q = 0; q < IX_FB; q++) {
                                const bool g = off[q] != 0xFFFFFFFFu && off[q] < ix_row_x<CSR, W>(p, xrow, scol, e0, n, c[q], samp, ns, sd, bm, pre);
                                const unsigned gm = __ballot_sync(FULL, g);
                                if (gm) {
                                    if (lane == 0) h[jq[q]] = t0 + __ffs(gm) - 1;
                                    live &= ~(1u << q);
                                }
                            }
                        }
#pragma unroll
                        for (int q = 0; q < IX_FB; q++)
                            if (((live >> q) & 1u) && lane == 0) h[jq[q]] = IX_SAT;   // no green draw before the cap
                    }
                    }
                    __syncthreads();
                    if (s_nu <= (uint32_t)CAPR) break;
                }
            }
        }
        __syncthreads();
        if (p.plan && threadIdx.x == 0) p.plan[row] = (uint8_t)plan;
        // ---- a9: h = t + 1, or the cap
        using sig_t = typename std::conditional<SIGB == 1, uint8_t, uint16_t>::type;
        sig_t *out = reinterpret_cast<sig_t *>(p.sig) + row * (int64_t)p.k;
        for (uint32_t j = threadIdx.x; j < p.k; j += NT) {
            const uint32_t v = h[j];
            const bool s = v >= IX_SAT;
            sat += s;
            out[j] = (sig_t)(s ? p.cap : v + 1);
        }
    }
    if (p.n_sat) {
#pragma unroll
        for (int o = 16; o; o >>= 1) sat += __shfl_xor_sync(FULL, sat, o);
        if (lane == 0 && sat) atomicAdd(p.n_sat, sat);
    }
}

template <int SIGB, bool CSR, int NW, typename W>
static wmh_status ix_launch(IxParams p, cudaStream_t s) {
    auto kern = hash_index_kernel<SIGB, CSR, NW, W>;
    int dev = 0, smem_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
    // stage CSR columns while 2048/(32*NW) rows still fit per SM
    if (CSR) {
        const int rows_sm = 2048 / (32 * NW);
        const int64_t budget = (int64_t)smem_sm / rows_sm - 1024 - (int64_t)p.k * 4 - (int64_t)(2 * NW * 32 * 8 + 33) * 4;
        p.capn = (int)std::max<int64_t>(0, std::min<int64_t>(8192, budget / 4));
    } else {
        // the dense row staged as words for the fallback lookups, when short
        // (measured: 4 KiB rows cost more in occupancy than they save)
        static const int stage_max = getenv("WMH_INDEX_STAGE_MAX") ? atoi(getenv("WMH_INDEX_STAGE_MAX")) : 1024;
        p.capn = p.D <= stage_max ? (int)((p.D * (int64_t)sizeof(W) + 3) / 4) : 0;
    }
    const size_t smem = (size_t)p.k * 4 + (size_t)(2 * NW * 32 * 8 + 33) * 4 + (size_t)p.capn * 4;
    {
        int optin = 0;
        cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
        if (smem > (size_t)optin) { set_error("wmh_hash: k=%u needs %zu B of shared memory per row", p.k, smem); return WMH_EINVAL; }
    }
    WMH_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem), "index smem attr");
    int per_sm = 0;
    WMH_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NW * 32, smem), "index occupancy");
    if (per_sm < 1) { set_error("wmh_hash: k=%u needs %zu B of shared memory per row", p.k, smem); return WMH_EINVAL; }
    const int64_t grid = std::min<int64_t>((int64_t)num_sms() * per_sm, p.n_rows);
    kernel_timer_begin(s);
    kern<<<(unsigned)grid, NW * 32, smem, s>>>(p);
    kernel_timer_end(s);
    WMH_LAUNCH_CHECK("hash_index launch");
    if (getenv("WMH_INDEX_STATS")) {
        fprintf(stderr, "[wmh index] NW=%d per_sm=%d grid=%lld capn=%d E=%d B=", NW, per_sm, (long long)grid, p.capn,
                p.ep.E);
        for (int e = 1; e <= p.ep.E; e++) fprintf(stderr, "%u%s", p.ep.B[e], e < p.ep.E ? "," : "\n");
    }
    return WMH_OK;
}

template <int SIGB, bool CSR, typename W>
static wmh_status ix_launch_nw(const IxParams &p, int nw, cudaStream_t s) {
    switch (nw) {
        case 1: return ix_launch<SIGB, CSR, 1, W>(p, s);
        case 2: return ix_launch<SIGB, CSR, 2, W>(p, s);
        case 4: return ix_launch<SIGB, CSR, 4, W>(p, s);
        default: return ix_launch<SIGB, CSR, 8, W>(p, s);
    }
}

template <int SIGB, bool CSR>
static wmh_status ix_launch_w(const IxParams &p, int nw, int wb, cudaStream_t s) {
    return wb == 2 ? ix_launch_nw<SIGB, CSR, uint16_t>(p, nw, s) : ix_launch_nw<SIGB, CSR, uint8_t>(p, nw, s);
}

// Index horizon T: draws t < T are filed.  0 = automatic: from the layout's
// row-sum statistics (the 0.1% quantile s_q of prepare's rows) T covers
// ln(4k) / s_q draws, i.e. the k hashes of a row at s_q almost all resolve in
// the index; without statistics T = cap.
uint32_t index_horizon(const wmh_layout *L, uint32_t k, uint32_t cap, uint32_t hint) {
    uint64_t T = hint ? hint : cap;
    if (!hint && L->rowsum_q > 0) {
        const double s = std::min(0.999, (double)L->rowsum_q / (double)L->M);
        T = (uint64_t)ceil(log(4.0 * k) / -log1p(-s));
    }
    T = std::max<uint64_t>(1, std::min<uint64_t>(T, cap));
    const uint64_t max_entries = 1ull << 29;     // nested epochs hold <= 4/3 k T entries
    if ((uint64_t)k * T > max_entries) T = std::max<uint64_t>(1, max_entries / k);
    return (uint32_t)T;
}

static IxEpochs index_epochs(uint32_t T) {
    IxEpochs ep;
    ep.B[0] = 0;
    int E = 0;
    // x2 steps up to 512 draws (dense rows at s ~ 0.05 stop there), x4 beyond
    static const uint64_t x2max = getenv("WMH_INDEX_X2MAX") ? (uint64_t)atoll(getenv("WMH_INDEX_X2MAX")) : 512;
    for (uint64_t b = 32; b < T && E < IX_MAXE - 1; b *= (b < x2max ? 2 : 4)) ep.B[++E] = (uint32_t)b;
    // a last step shorter than half the previous boundary is merged into it
    if (E > 0 && (uint64_t)T * 2 < (uint64_t)ep.B[E] * 3) E--;
    ep.B[++E] = T;
    ep.E = E;
    for (int i = E + 1; i <= IX_MAXE; i++) ep.B[i] = T;
    return ep;
}

// The largest k the rows kernel takes: its shared memory holds h[k] (4 B per
// hash) next to the 8-warp range buffers; also bounded by the 16-bit j of an entry.
uint32_t index_k_max() {
    static uint32_t kmax = 0;
    if (!kmax) {
        int dev = 0, optin = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
        const int64_t fixed = (int64_t)(2 * 8 * 32 * 8 + 33) * 4 + 256;     // + the static shared variables
        kmax = (uint32_t)std::max<int64_t>(1, std::min<int64_t>(65536, ((int64_t)optin - fixed) / 4));
    }
    return kmax;
}

// Can the index be built for (layout, k, cap, horizon)?  k within index_k_max(),
// fewer than 2^32 filed instances, and a key space E*M the direct partition
// covers (<= 16383 chunks of <= 2^15 cells).  AUTO only picks the index when so.
bool index_feasible(const wmh_layout *L, uint32_t k, uint32_t cap, uint32_t horizon) {
    if (k > index_k_max()) return false;
    const IxEpochs ep = index_epochs(index_horizon(L, k, cap, horizon));
    uint64_t n_inst = 0;
    for (int e = 0; e < ep.E; e++) n_inst += (uint64_t)k * ep.B[e + 1];
    return n_inst < (1ull << 32) && (uint64_t)ep.E * L->M <= 16383ull * 32768ull;
}

wmh_status index_build(const HashArgs &a, uint32_t horizon, IndexBuilt *out) {
    *out = IndexBuilt();
    if (a.k > index_k_max()) {
        set_error("wmh_hash: the index kernel takes k <= %u (h[k] in shared memory)", index_k_max());
        return WMH_EINVAL;
    }
    const wmh_layout *L = a.L;
    const uint32_t M = (uint32_t)L->M;
    const uint32_t T = index_horizon(L, a.k, a.cap, horizon);
    const IxEpochs ep = index_epochs(T);

    IxBuild b;
    b.S = a.S;
    b.k = a.k;
    b.T = T;
    b.M = M;
    b.ep = ep;
    b.n_keys = (uint64_t)ep.E * M;
    b.n_draws = (uint64_t)a.k * T;
    uint64_t n_inst = 0;
    for (int e = 0; e < ep.E; e++) n_inst += (uint64_t)a.k * ep.B[e + 1];
    if (n_inst >= (1ull << 32)) { set_error("wmh_hash: index too large (k*T)"); return WMH_EINVAL; }
    const int sms = num_sms();
    // chunks of ~equal entry counts: epoch e holds k*B[e+1]/M entries per cell
    // in expectation (the cells are equiprobable), so its chunks span
    // 2^cb[e] ~ target / density cells; <= 16383 chunks (the partition's
    // shared cursors), <= 2^15 cells per chunk (the sort's shared histogram).
    // Fewer, larger chunks measured faster (the partition's scattered stores
    // dominate): target = n_inst / 1000 (c3: 2.7 ms build, c4: 8.1 ms)
    static const double chunks_env = getenv("WMH_INDEX_CHUNKS") ? atof(getenv("WMH_INDEX_CHUNKS")) : 0.0;
    for (double target = std::max(4096.0, (double)n_inst / (chunks_env > 0 ? chunks_env : 1000.0));; target *= 2) {
        uint64_t nc = 0;
        b.cb_max = 0;
        for (int e = 0; e < ep.E; e++) {
            const double dens = (double)a.k * ep.B[e + 1] / (double)M;
            int cb = (int)floor(log2(std::max(1.0, target / dens)));
            cb = std::max(6, std::min(15, cb));
            b.cb[e] = cb;
            b.cb_max = std::max(b.cb_max, cb);
            b.cbase[e] = (uint32_t)nc;
            nc += ((uint64_t)M + (1ull << cb) - 1) >> cb;
        }
        b.cbase[ep.E] = (uint32_t)nc;
        if (nc <= 16383) { b.n_chunks = (uint32_t)nc; break; }
        if (target > 1e12) { set_error("wmh_hash: index key space too large (E*M = %llu)", (unsigned long long)b.n_keys); return WMH_EINVAL; }
    }
    b.n_cta = (int)std::max<uint64_t>(1, std::min<uint64_t>((uint64_t)sms * 2, (b.n_draws + 4095) / 4096));
    b.per_cta = (b.n_draws + b.n_cta - 1) / b.n_cta;

    const uint64_t n_h = (uint64_t)b.n_chunks * b.n_cta + 1;
    const int64_t nt = (int64_t)((n_h + SC_TILE - 1) / SC_TILE);
    auto al = [](uint64_t v) { return (v + 255) & ~(uint64_t)255; };
    const uint64_t pos_b = al((b.n_keys + 1) * 4), vals_b = al(n_inst * 4), tmp_b = al(n_inst * 4),
                   h_b = al(n_h * 4), sums_b = al((uint64_t)nt * 4 + 4), tab_b = al((uint64_t)a.k * T0 * 8),
                   cs_b = (L->flags & WMH_LAYOUT_UNIFORM) ? al((uint64_t)ep.E * (L->dim + 1) * 4) : 0;
    uint8_t *scr = nullptr;
    WMH_CUDA_TRY(cudaMallocAsync((void **)&scr, pos_b + vals_b + tmp_b + h_b + sums_b + tab_b + cs_b + 256, a.stream),
                 "index alloc");
    uint32_t *pos = reinterpret_cast<uint32_t *>(scr);
    uint32_t *vals = reinterpret_cast<uint32_t *>(scr + pos_b);
    uint32_t *tmp = reinterpret_cast<uint32_t *>(scr + pos_b + vals_b);
    uint32_t *H = reinterpret_cast<uint32_t *>(scr + pos_b + vals_b + tmp_b);
    uint32_t *sums = reinterpret_cast<uint32_t *>(scr + pos_b + vals_b + tmp_b + h_b);
    uint2 *table = reinterpret_cast<uint2 *>(scr + pos_b + vals_b + tmp_b + h_b + sums_b);
    uint32_t *colstart = reinterpret_cast<uint32_t *>(scr + pos_b + vals_b + tmp_b + h_b + sums_b + tab_b);
    unsigned long long *ctr = reinterpret_cast<unsigned long long *>(scr + pos_b + vals_b + tmp_b + h_b + sums_b + tab_b + cs_b);
    wmh_status st = WMH_OK;
    do {
        if (cudaMemsetAsync(H, 0, 4, a.stream) != cudaSuccess || cudaMemsetAsync(ctr, 0, 8, a.stream) != cudaSuccess) {
            st = cuda_fail(cudaGetLastError(), "index memset");
            break;
        }
        static const int build_env = getenv("WMH_INDEX_BUILD") ? atoi(getenv("WMH_INDEX_BUILD")) : 2;
        st = build_env != 1 ? index_build_sorted(a.S, a.k, M, ep, pos, vals, a.stream) : WMH_EINVAL;
        if (st != WMH_OK && st != WMH_EINVAL) break;
        if (st == WMH_OK) {                      // the coalesced build (index_build.cu)
        } else {                                 // the direct partition (very wide key spaces)
        st = WMH_OK;
        const size_t psm = (size_t)b.n_chunks * 4;
        cudaFuncSetAttribute(ix_partition<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)psm);
        cudaFuncSetAttribute(ix_partition<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)psm);
        ix_partition<false><<<b.n_cta, 512, psm, a.stream>>>(b, H, tmp);
        count_launch();
        if (cudaGetLastError() != cudaSuccess) { st = cuda_fail(cudaGetLastError(), "index count"); break; }
        if ((st = scan_u32_inplace(H + 1, (int64_t)(n_h - 1), sums, a.stream)) != WMH_OK) break;
        ix_partition<true><<<b.n_cta, 512, psm, a.stream>>>(b, H, tmp);
        count_launch();
        if (cudaGetLastError() != cudaSuccess) { st = cuda_fail(cudaGetLastError(), "index partition"); break; }
        const size_t csm = (size_t)4 << b.cb_max;
        cudaFuncSetAttribute(ix_chunk_sort, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)csm);
        ix_chunk_sort<<<b.n_chunks, SC_T, csm, a.stream>>>(b, H, tmp, pos, vals);
        count_launch();
        if (cudaGetLastError() != cudaSuccess) { st = cuda_fail(cudaGetLastError(), "index sort"); break; }
        }

        const uint32_t uni = (L->flags & WMH_LAYOUT_UNIFORM) ? L->uniform_m : 0u;
        const uint32_t *pk = (L->flags & WMH_LAYOUT_WIDE) ? nullptr : L->cell_pack;
        if ((st = launch_draw_table(table, a.k, a.S, M, pk, uni, 1u, a.stream, L->int_to_comp, L->comp_to_m)) != WMH_OK) break;
        if (uni) {                               // uniform bounds only (the row kernel's lookup)
            const int64_t total = (int64_t)ep.E * (L->dim + 1);
            const int blocks = (int)std::min<int64_t>((int64_t)sms * 8, (total + 255) / 256);
            ix_colstart_kernel<<<blocks, 256, 0, a.stream>>>(pos, L->comp_to_m, uni, ep.E, M, L->dim, colstart);
            count_launch();
            if (cudaGetLastError() != cudaSuccess) { st = cuda_fail(cudaGetLastError(), "index colstart"); break; }
        }

    } while (0);
    if (st != WMH_OK) {
        cudaFreeAsync(scr, a.stream);
        return st;
    }
    out->scr = scr;
    out->pos = pos;
    out->colstart = colstart;
    out->vals = vals;
    out->table = table;
    out->ctr = ctr;
    out->ep = ep;
    out->T = T;
    return WMH_OK;
}

void index_free(IndexBuilt &ix, cudaStream_t s) {
    if (ix.scr) cudaFreeAsync(ix.scr, s);
    ix = IndexBuilt();
}

wmh_status index_rows(const HashArgs &a, const IndexBuilt &ix) {
    const wmh_layout *L = a.L;
    const uint32_t M = (uint32_t)L->M;
    if (a.rows.n_rows == 0) return WMH_OK;
    // a row counter of this call's own (stream-ordered): two runs of one index
    // on different streams must not share the work-stealing counter
    unsigned long long *ctr = nullptr;
    WMH_CUDA_TRY(cudaMallocAsync((void **)&ctr, 8, a.stream), "index row counter alloc");
    if (cudaMemsetAsync(ctr, 0, 8, a.stream) != cudaSuccess) { cudaFreeAsync(ctr, a.stream); return cuda_fail(cudaGetLastError(), "index row counter"); }
    wmh_status st = WMH_OK;
    const uint32_t *pos = ix.pos, *vals = ix.vals;
    const uint2 *table = ix.table;
    const IxEpochs ep = ix.ep;
    IxParams p;
    const bool csr = a.rows.kind == WMH_CSR;
    p.x = a.rows.dense;
    p.row_ptr = a.rows.row_ptr;
    p.col = a.rows.col;
    p.val = a.rows.val;
    p.n_rows = a.rows.n_rows;
    p.D = a.rows.dim;
    p.comp_to_m = L->comp_to_m;
    p.pack = (L->flags & WMH_LAYOUT_WIDE) ? nullptr : L->cell_pack;
    p.i2c = L->int_to_comp;
    p.uni_m = (L->flags & WMH_LAYOUT_UNIFORM) ? L->uniform_m : 0u;
    p.M = M;
    p.pos = pos;
    p.colstart = ix.colstart;
    p.vals = vals;
    p.table = table;
    p.ep = ep;
    p.S = a.S;
    p.k = a.k;
    p.cap = a.cap;
    p.capn = 0;
    // warps per row: >= 2; keep <= ~128 KiB of h[] per SM at 64 resident warps
    static const int nw_env = getenv("WMH_INDEX_NW") ? atoi(getenv("WMH_INDEX_NW")) : 0;
    int nw = 2;
    while (nw < 8 && (uint64_t)(64 / nw) * a.k * 4 > (128u << 10)) nw *= 2;
    if (nw_env == 1 || nw_env == 2 || nw_env == 4 || nw_env == 8) nw = nw_env;
    // the plan's cost of one fallback draw in units of one index entry: an
    // unstaged CSR row's x_c lookup is a binary search over the row's columns in
    // global memory (~11 dependent loads) with 1-4 warps, a shared-memory search of
    // a column sample plus one or two loads with 8 (measured sweeps: c3 at 2 warps
    // 10.07 ms at 16, 9.61 at 64-100; c4 at 8 warps 18.27 at 16, 18.19 at 24-32)
    static const float cfs = getenv("WMH_INDEX_CF") ? (float)atof(getenv("WMH_INDEX_CF")) : 0.f;
    p.cf_dense = cfs > 0 ? cfs : 2.f;
    p.cf_smem = cfs > 0 ? cfs : 3.f;
    p.cf_global = cfs > 0 ? cfs : (nw == 8 ? 24.f : 64.f);
    // 8 warps, CSR: the row's column bitmap (ceil(D/32) words) + the first-column
    // index per word (uint16) + the uint16 hash list must fit the 2*CAPR + 33 words
    // of the range buffers (D <= ~66,000); WMH_INDEX_BITMAP=0 turns it off
    static const int bm_env = getenv("WMH_INDEX_BITMAP") ? atoi(getenv("WMH_INDEX_BITMAP")) : 1;
    static const float cfb = getenv("WMH_INDEX_CF_BM") ? (float)atof(getenv("WMH_INDEX_CF_BM")) : 0.f;
    {
        constexpr int64_t capr8 = 8 * 32 * 8;
        const int64_t bmw = (a.rows.dim + 31) / 32;
        p.bm_words = (csr && nw == 8 && bm_env && bmw + (bmw + 1) / 2 + capr8 / 2 <= 2 * capr8 + 33) ? (int)bmw : 0;
    }
    p.cf_bitmap = cfs > 0 ? cfs : cfb > 0 ? cfb : 6.f;
    p.sig = a.sig;
    p.n_sat = a.n_sat;
    p.row_ctr = ctr;
    p.perm = nullptr;
    p.plan = reinterpret_cast<uint8_t *>(a.plan_out);
    // processing order by planned epoch when the per-cell tables are far larger
    // than L2 (measured: c4's 535 MB pos[] 22.8 -> 20.2 ms; c3's 194 MB and c2r
    // gain nothing and pay the pre-pass); WMH_INDEX_ORDER=0/1 forces it off/on
    static const int order_env = getenv("WMH_INDEX_ORDER") ? atoi(getenv("WMH_INDEX_ORDER")) : -1;
    int l2 = 0, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev);
    const bool big_tables = (uint64_t)ep.E * M * 4 > 3ull * (uint64_t)l2;
    uint8_t *oscr = nullptr;
    if ((order_env == 1 || (order_env < 0 && big_tables)) && a.rows.n_rows >= 4096 && a.rows.n_rows < (1ll << 32)) {
        const size_t pe_b = ((size_t)a.rows.n_rows + 255) & ~(size_t)255, pm_b = (size_t)a.rows.n_rows * 4;
        if (cudaMallocAsync((void **)&oscr, pe_b + pm_b + 2 * IX_MAXE * 4 + 256, a.stream) != cudaSuccess) {
            cudaFreeAsync(ctr, a.stream);
            return cuda_fail(cudaGetLastError(), "index order alloc");
        }
        uint8_t *row_epoch = oscr;
        uint32_t *perm = reinterpret_cast<uint32_t *>(oscr + pe_b);
        unsigned int *cnt = reinterpret_cast<unsigned int *>(oscr + pe_b + ((pm_b + 255) & ~(size_t)255));
        unsigned int *cursor = cnt + IX_MAXE;
        if (cudaMemsetAsync(cnt, 0, 2 * IX_MAXE * 4, a.stream) != cudaSuccess) {
            cudaFreeAsync(oscr, a.stream);
            cudaFreeAsync(ctr, a.stream);
            return cuda_fail(cudaGetLastError(), "index order memset");
        }
        const int blocks = (int)std::min<int64_t>((int64_t)num_sms() * 8, (a.rows.n_rows * 32 + 255) / 256);
        const int wbo = weight_bytes(a.rows);
        if (csr) {
            if (wbo == 2) ix_order_count<true, uint16_t><<<blocks, 256, 0, a.stream>>>(p, row_epoch, cnt);
            else ix_order_count<true, uint8_t><<<blocks, 256, 0, a.stream>>>(p, row_epoch, cnt);
        } else {
            if (wbo == 2) ix_order_count<false, uint16_t><<<blocks, 256, 0, a.stream>>>(p, row_epoch, cnt);
            else ix_order_count<false, uint8_t><<<blocks, 256, 0, a.stream>>>(p, row_epoch, cnt);
        }
        count_launch();
        const int sblocks = (int)std::min<int64_t>((int64_t)num_sms() * 8, (a.rows.n_rows + 255) / 256);
        ix_order_scatter<<<sblocks, 256, 0, a.stream>>>(a.rows.n_rows, ep.E, row_epoch, cnt, cursor, perm);
        count_launch();
        if (cudaGetLastError() != cudaSuccess) { cudaFreeAsync(oscr, a.stream); cudaFreeAsync(ctr, a.stream); return cuda_fail(cudaGetLastError(), "index order"); }
        p.perm = perm;
    }
    const int wb = weight_bytes(a.rows);
    if (a.sig_bytes == 1) st = csr ? ix_launch_w<1, true>(p, nw, wb, a.stream) : ix_launch_w<1, false>(p, nw, wb, a.stream);
    else st = csr ? ix_launch_w<2, true>(p, nw, wb, a.stream) : ix_launch_w<2, false>(p, nw, wb, a.stream);
    if (oscr) cudaFreeAsync(oscr, a.stream);
    cudaFreeAsync(ctr, a.stream);
    return st;
}

wmh_status launch_hash_index(const HashArgs &a, uint32_t horizon) {
    IndexBuilt ix;
    wmh_status st = index_build(a, horizon, &ix);
    if (st != WMH_OK) return st;
    st = index_rows(a, ix);
    index_free(ix, a.stream);
    return st;
}

}  // namespace wmh
