// index_build.cu -- the INDEX kernel's build with coalesced stores (the
// default; hash_index.cu keeps the direct partition as WMH_INDEX_BUILD=1).
//
// Same output as the direct build -- epoch e's draws t < B[e+1] of every hash,
// sorted by cell, pos[e*M + r] = first entry of cell r -- but every store of
// the 4-byte entries is a run written by consecutive threads:
//   A  count the instances (epoch, j, t) per chunk and per super-chunk (32
//      consecutive chunks of one epoch), per CTA slice of the instance space
//   B  each CTA sorts a batch of 8192 instances by super-chunk in shared memory
//      and writes every super-chunk's run at its cursor (runs of ~10)
//   C  one CTA per super-chunk sorts its entries by chunk in shared-memory
//      batches and writes runs into the chunks (runs of ~250)
//   D  one CTA per chunk counting-sorts its (<= 8192) entries by cell in
//      shared memory, writes pos[] of its cells and the sorted entries at once
// The instance space is flat: epoch e holds k * B[e+1] instances (j, t < B[e+1]),
// and an instance's cell is re-drawn from (j, t) wherever it is needed.
#include <algorithm>

#include "common.cuh"

namespace wmh {

constexpr int X3_T = 1024;                      // threads per CTA
constexpr int X3_NB = 8192;                     // instances per batch (8 per thread)
constexpr int X3_GS = 32;                       // chunks per super-chunk
constexpr int X3_CAP = 8192;                    // entries a chunk sorts in shared memory
constexpr int X3_CBMAX = 13;                    // log2 of the most cells per chunk

struct X3Params {
    uint64_t S;
    uint32_t k, M;
    int E;
    uint32_t B[IX_MAXE + 1];
    uint64_t ibase[IX_MAXE + 1];                // first flat instance of epoch e
    int cb[IX_MAXE];                            // log2 cells per chunk in epoch e
    uint32_t cbase[IX_MAXE + 1];                // first chunk of epoch e
    uint32_t sbase[IX_MAXE + 1];                // first super-chunk of epoch e
    uint32_t n_chunks, n_super;
    uint64_t n_inst, n_keys;
    uint64_t per_cta;
    int n_cta;
};

struct X3Inst {
    uint32_t val;                               // (j << 16) | t
    uint32_t r;                                 // cell
    int e;
};

// instance i (a thread visits increasing i: e advances from the previous call's)
__device__ __forceinline__ X3Inst x3_inst(const X3Params &p, uint64_t i, int &e) {
    while (e + 1 < p.E && i >= p.ibase[e + 1]) e++;
    const uint32_t w = (uint32_t)(i - p.ibase[e]);     // < k * B[e+1] <= 2^16 * 2^16
    const uint32_t Bn = p.B[e + 1];
    const uint32_t j = w / Bn, t = w - j * Bn;
    X3Inst o;
    o.val = (j << 16) | t;
    o.r = mulhi_range(splitmix64(p.S ^ ((uint64_t)j << 32) ^ (uint64_t)t), p.M);
    o.e = e;
    return o;
}

__device__ __forceinline__ uint32_t x3_redraw(const X3Params &p, uint32_t val) {
    return mulhi_range(splitmix64(p.S ^ ((uint64_t)(val >> 16) << 32) ^ (uint64_t)(val & 0xFFFFu)), p.M);
}

// block-wide exclusive scan (X3_T threads), *total optional
__device__ __forceinline__ uint32_t x3_excl_scan(uint32_t v, uint32_t *total) {
    __shared__ uint32_t ws[X3_T / 32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t u = __shfl_up_sync(0xFFFFFFFFu, incl, o);
        if (lane >= o) incl += u;
    }
    if (lane == 31) ws[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        const uint32_t w = ws[lane];
        uint32_t wi = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t u = __shfl_up_sync(0xFFFFFFFFu, wi, o);
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

// exclusive scan of cnt[0..n) in place (n <= X3_T * per), returns the total
__device__ __forceinline__ uint32_t x3_scan_array(uint32_t *cnt, uint32_t n) {
    __shared__ uint32_t tot;
    const uint32_t per = (n + X3_T - 1) / X3_T, i0 = threadIdx.x * per, i1 = min(n, i0 + per);
    uint32_t s = 0;
    for (uint32_t i = i0; i < i1; i++) s += cnt[i];
    uint32_t run = x3_excl_scan(s, &tot);
    for (uint32_t i = i0; i < i1; i++) {
        const uint32_t v = cnt[i];
        cnt[i] = run;
        run += v;
    }
    __syncthreads();
    return tot;
}

// A: per-chunk totals (global atomics, one per nonzero counter per CTA) and
// per-(super-chunk, CTA) counts
__global__ void __launch_bounds__(X3_T) x3_count(const X3Params p, uint32_t *__restrict__ chunk_cnt,
                                                 uint32_t *__restrict__ Hs) {
    extern __shared__ uint32_t sm[];
    uint32_t *cc = sm;                          // [n_chunks]
    uint32_t *sc = sm + p.n_chunks;             // [n_super]
    for (uint32_t i = threadIdx.x; i < p.n_chunks + p.n_super; i += X3_T) sm[i] = 0;
    __syncthreads();
    const uint64_t i0 = (uint64_t)blockIdx.x * p.per_cta, i1 = min(p.n_inst, i0 + p.per_cta);
    int ee = 0;
    for (uint64_t i = i0 + threadIdx.x; i < i1; i += X3_T) {
        const X3Inst x = x3_inst(p, i, ee);
        const uint32_t loc = x.r >> p.cb[x.e];
        atomicAdd(cc + p.cbase[x.e] + loc, 1u);
        atomicAdd(sc + p.sbase[x.e] + loc / X3_GS, 1u);
    }
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < p.n_chunks; i += X3_T)
        if (cc[i]) atomicAdd(chunk_cnt + 1 + i, cc[i]);
    for (uint32_t s = threadIdx.x; s < p.n_super; s += X3_T) Hs[1 + (uint64_t)s * p.n_cta + blockIdx.x] = sc[s];
}

// B: batches sorted by super-chunk in shared memory, runs written at the cursors
__global__ void __launch_bounds__(X3_T) x3_partition(const X3Params p, const uint32_t *__restrict__ Hs,
                                                     uint32_t *__restrict__ tmp1) {
    extern __shared__ uint32_t sm[];
    uint32_t *cur = sm;                         // [n_super] global write cursor of this CTA
    uint32_t *cnt = cur + p.n_super;            // [n_super] batch counts -> batch starts
    uint32_t *rnk = cnt + p.n_super;            // [n_super] running rank while scattering
    uint32_t *sv = rnk + p.n_super;             // [X3_NB] staged entries
    uint32_t *ss = sv + X3_NB;                  // [X3_NB] their super-chunks
    for (uint32_t s = threadIdx.x; s < p.n_super; s += X3_T) cur[s] = Hs[(uint64_t)s * p.n_cta + blockIdx.x];
    const uint64_t i0 = (uint64_t)blockIdx.x * p.per_cta, i1 = min(p.n_inst, i0 + p.per_cta);
    int ee = 0;
    for (uint64_t b0 = i0; b0 < i1; b0 += X3_NB) {
        const uint32_t nb = (uint32_t)min((uint64_t)X3_NB, i1 - b0);
        for (uint32_t s = threadIdx.x; s < p.n_super; s += X3_T) cnt[s] = 0;
        __syncthreads();
        uint32_t myv[X3_NB / X3_T], mys[X3_NB / X3_T];
#pragma unroll
        for (int q = 0; q < X3_NB / X3_T; q++) {
            const uint32_t li = threadIdx.x + q * X3_T;
            mys[q] = 0xFFFFFFFFu;
            if (li < nb) {
                const X3Inst x = x3_inst(p, b0 + li, ee);
                myv[q] = x.val;
                mys[q] = p.sbase[x.e] + (x.r >> p.cb[x.e]) / X3_GS;
                atomicAdd(cnt + mys[q], 1u);
            }
        }
        __syncthreads();
        x3_scan_array(cnt, p.n_super);          // batch start of each super-chunk
        for (uint32_t s = threadIdx.x; s < p.n_super; s += X3_T) rnk[s] = cnt[s];
        __syncthreads();
#pragma unroll
        for (int q = 0; q < X3_NB / X3_T; q++)
            if (mys[q] != 0xFFFFFFFFu) {
                const uint32_t d = atomicAdd(rnk + mys[q], 1u);
                sv[d] = myv[q];
                ss[d] = mys[q];
            }
        __syncthreads();
        for (uint32_t li = threadIdx.x; li < nb; li += X3_T) {      // runs: consecutive threads, one super
            const uint32_t s = ss[li];
            tmp1[cur[s] + (li - cnt[s])] = sv[li];
        }
        __syncthreads();
        for (uint32_t s = threadIdx.x; s < p.n_super; s += X3_T) cur[s] += rnk[s] - cnt[s];
        __syncthreads();
    }
}

// C: one CTA per super-chunk: entries into their chunks (runs via a shared sort)
__global__ void __launch_bounds__(X3_T) x3_superchunk(const X3Params p, const uint32_t *__restrict__ Hs,
                                                      const uint32_t *__restrict__ chunk_start,
                                                      const uint32_t *__restrict__ tmp1, uint32_t *__restrict__ tmp2) {
    __shared__ uint32_t cur[X3_GS], cnt[X3_GS], rnk[X3_GS];
    __shared__ uint32_t sv[X3_NB];
    __shared__ uint8_t sl[X3_NB];
    const uint32_t s = blockIdx.x;
    int e = 0;
    for (int q = 1; q < p.E; q++)
        if (s >= p.sbase[q]) e = q;
    const uint32_t c0 = p.cbase[e] + (s - p.sbase[e]) * X3_GS;     // first chunk of this super-chunk
    const uint32_t nck = min((uint32_t)X3_GS, p.cbase[e + 1] - c0);
    const uint32_t beg = Hs[(uint64_t)s * p.n_cta], end = Hs[(uint64_t)(s + 1) * p.n_cta];
    if (threadIdx.x < X3_GS) cur[threadIdx.x] = threadIdx.x < nck ? chunk_start[c0 + threadIdx.x] : 0u;
    const int cb = p.cb[e];
    for (uint32_t b0 = beg; b0 < end; b0 += X3_NB) {
        const uint32_t nb = min((uint32_t)X3_NB, end - b0);
        if (threadIdx.x < X3_GS) cnt[threadIdx.x] = 0;
        __syncthreads();
        uint32_t myv[X3_NB / X3_T], myl[X3_NB / X3_T];
#pragma unroll
        for (int q = 0; q < X3_NB / X3_T; q++) {
            const uint32_t li = threadIdx.x + q * X3_T;
            myl[q] = 0xFFFFFFFFu;
            if (li < nb) {
                myv[q] = tmp1[b0 + li];
                myl[q] = (x3_redraw(p, myv[q]) >> cb) - (c0 - p.cbase[e]);
                atomicAdd(cnt + myl[q], 1u);
            }
        }
        __syncthreads();
        if (threadIdx.x < 32) {                 // exclusive scan of the 32 chunk counts
            const uint32_t v = cnt[threadIdx.x];
            uint32_t incl = v;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t u = __shfl_up_sync(0xFFFFFFFFu, incl, o);
                if ((int)threadIdx.x >= o) incl += u;
            }
            cnt[threadIdx.x] = incl - v;
            rnk[threadIdx.x] = incl - v;
        }
        __syncthreads();
#pragma unroll
        for (int q = 0; q < X3_NB / X3_T; q++)
            if (myl[q] != 0xFFFFFFFFu) {
                const uint32_t d = atomicAdd(rnk + myl[q], 1u);
                sv[d] = myv[q];
                sl[d] = (uint8_t)myl[q];
            }
        __syncthreads();
        for (uint32_t li = threadIdx.x; li < nb; li += X3_T) {
            const uint32_t l = sl[li];
            tmp2[cur[l] + (li - cnt[l])] = sv[li];
        }
        __syncthreads();
        if (threadIdx.x < X3_GS) cur[threadIdx.x] += rnk[threadIdx.x] - cnt[threadIdx.x];
        __syncthreads();
    }
}

// D: one CTA per chunk: counting sort by cell in shared memory
__global__ void __launch_bounds__(X3_T) x3_chunksort(const X3Params p, const uint32_t *__restrict__ chunk_start,
                                                     const uint32_t *__restrict__ tmp2, uint32_t *__restrict__ pos,
                                                     uint32_t *__restrict__ vals) {
    extern __shared__ uint32_t sm[];
    const uint32_t c = blockIdx.x;
    int e = 0;
    for (int q = 1; q < p.E; q++)
        if (c >= p.cbase[q]) e = q;
    const int cb = p.cb[e];
    const uint32_t r0 = (c - p.cbase[e]) << cb;
    const uint32_t nloc = min(1u << cb, p.M - r0);
    const uint32_t beg = chunk_start[c], end = chunk_start[c + 1], n = end - beg;
    const bool fits = n <= (uint32_t)X3_CAP;
    uint32_t *cnt = sm;                         // [2^cb]
    uint32_t *in = sm + (1u << cb);             // [X3_CAP] entries (fits) ...
    uint32_t *out = in + X3_CAP;                // [X3_CAP] ... sorted
    for (uint32_t i = threadIdx.x; i < nloc; i += X3_T) cnt[i] = 0;
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < n; i += X3_T) {
        const uint32_t v = tmp2[beg + i];
        if (fits) in[i] = v;
        atomicAdd(cnt + (x3_redraw(p, v) - r0), 1u);
    }
    __syncthreads();
    x3_scan_array(cnt, nloc);                   // cnt[i] = entries of cells < i within the chunk
    const uint64_t key0 = (uint64_t)e * p.M + r0;
    for (uint32_t i = threadIdx.x; i < nloc; i += X3_T) pos[key0 + i] = beg + cnt[i];
    if (c + 1 == p.n_chunks && threadIdx.x == 0) pos[p.n_keys] = end;
    __syncthreads();
    if (fits) {
        for (uint32_t i = threadIdx.x; i < n; i += X3_T) {
            const uint32_t v = in[i];
            out[atomicAdd(cnt + (x3_redraw(p, v) - r0), 1u)] = v;
        }
        __syncthreads();
        for (uint32_t i = threadIdx.x; i < n; i += X3_T) vals[beg + i] = out[i];      // one coalesced run
    } else {                                    // rare oversized chunk: scatter straight to global
        for (uint32_t i = threadIdx.x; i < n; i += X3_T) {
            const uint32_t v = tmp2[beg + i];
            vals[beg + atomicAdd(cnt + (x3_redraw(p, v) - r0), 1u)] = v;
        }
    }
}

// Host side.  Writes pos (E*M + 1 words) and vals (n_inst words); scratch from
// the caller's stream-ordered pool.
wmh_status index_build_sorted(uint64_t S, uint32_t k, uint32_t M, const IxEpochs &ep, uint32_t *pos, uint32_t *vals,
                              cudaStream_t s) {
    X3Params p{};
    p.S = S;
    p.k = k;
    p.M = M;
    p.E = ep.E;
    for (int e = 0; e <= IX_MAXE; e++) p.B[e] = ep.B[e];
    uint64_t n_inst = 0;
    for (int e = 0; e < ep.E; e++) {
        p.ibase[e] = n_inst;
        n_inst += (uint64_t)k * ep.B[e + 1];
    }
    for (int e = ep.E; e <= IX_MAXE; e++) p.ibase[e] = n_inst;
    p.n_inst = n_inst;
    p.n_keys = (uint64_t)ep.E * M;
    // chunks of ~6K entries (the cells of epoch e are equiprobable: k*B[e+1]/M
    // entries each), at most 2^13 cells (the sort then runs 2 CTAs per SM);
    // super-chunks of 32 chunks of one epoch.  A target that needs too many
    // chunk counters doubles (chunks above X3_CAP entries sort through global
    // memory -- correct, slower); WMH_EINVAL asks the caller for the direct build.
    uint64_t nc = 0, ns = 0;
    for (double target = 6144.0;; target *= 2) {
        nc = ns = 0;
        for (int e = 0; e < ep.E; e++) {
            const double dens = (double)k * ep.B[e + 1] / (double)M;
            int cb = (int)floor(log2(std::max(1.0, target / dens)));
            cb = std::max(6, std::min(X3_CBMAX, cb));
            p.cb[e] = cb;
            p.cbase[e] = (uint32_t)nc;
            p.sbase[e] = (uint32_t)ns;
            const uint64_t ce = ((uint64_t)M + (1ull << cb) - 1) >> cb;
            nc += ce;
            ns += (ce + X3_GS - 1) / X3_GS;
        }
        if ((nc + ns) * 4 <= 180 * 1024) break;
        if (target > 1e9) {
            set_error("wmh_hash: index too wide for the sorted build (%llu chunks)", (unsigned long long)nc);
            return WMH_EINVAL;
        }
    }
    p.cbase[ep.E] = (uint32_t)nc;
    p.sbase[ep.E] = (uint32_t)ns;
    p.n_chunks = (uint32_t)nc;
    p.n_super = (uint32_t)ns;
    const int sms = num_sms();
    const size_t smA = ((size_t)nc + ns) * 4, smB = (size_t)ns * 12 + (size_t)X3_NB * 8;
    if (smB > 200 * 1024) {
        set_error("wmh_hash: index too wide for the sorted build (%llu super-chunks)", (unsigned long long)ns);
        return WMH_EINVAL;
    }
    p.n_cta = (int)std::max<uint64_t>(1, std::min<uint64_t>((uint64_t)sms * 2, (n_inst + X3_NB - 1) / X3_NB));
    p.per_cta = ((n_inst + p.n_cta - 1) / p.n_cta + X3_NB - 1) / X3_NB * X3_NB;

    auto al = [](uint64_t v) { return (v + 255) & ~(uint64_t)255; };
    const uint64_t n_hs = (uint64_t)ns * p.n_cta + 1;
    const uint64_t t_b = al(n_inst * 4), cc_b = al((nc + 2) * 4), hs_b = al(n_hs * 4);
    const uint64_t sums_b = al(((std::max<uint64_t>(n_hs, nc + 1) + 8191) / 8192 + 2) * 4);
    uint8_t *scr = nullptr;
    WMH_CUDA_TRY(cudaMallocAsync((void **)&scr, 2 * t_b + cc_b + hs_b + sums_b, s), "index build scratch");
    uint32_t *tmp1 = reinterpret_cast<uint32_t *>(scr);
    uint32_t *tmp2 = reinterpret_cast<uint32_t *>(scr + t_b);
    uint32_t *ccnt = reinterpret_cast<uint32_t *>(scr + 2 * t_b);
    uint32_t *Hs = reinterpret_cast<uint32_t *>(scr + 2 * t_b + cc_b);
    uint32_t *sums = reinterpret_cast<uint32_t *>(scr + 2 * t_b + cc_b + hs_b);
    wmh_status st = WMH_OK;
    do {
        if (cudaMemsetAsync(ccnt, 0, (nc + 2) * 4, s) != cudaSuccess || cudaMemsetAsync(Hs, 0, 4, s) != cudaSuccess) {
            st = cuda_fail(cudaGetLastError(), "index build memset");
            break;
        }
        cudaFuncSetAttribute(x3_count, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smA);
        x3_count<<<p.n_cta, X3_T, smA, s>>>(p, ccnt, Hs);
        count_launch();
        if (cudaGetLastError() != cudaSuccess) { st = cuda_fail(cudaGetLastError(), "index build count"); break; }
        // exclusive starts: ccnt[c] = entries of chunks < c (counts were added at +1)
        if ((st = scan_u32_inplace(ccnt + 1, (int64_t)nc, sums, s)) != WMH_OK) break;
        if ((st = scan_u32_inplace(Hs + 1, (int64_t)(n_hs - 1), sums, s)) != WMH_OK) break;
        cudaFuncSetAttribute(x3_partition, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smB);
        x3_partition<<<p.n_cta, X3_T, smB, s>>>(p, Hs, tmp1);
        count_launch();
        x3_superchunk<<<p.n_super, X3_T, 0, s>>>(p, Hs, ccnt, tmp1, tmp2);
        count_launch();
        int cbm = 0;
        for (int e = 0; e < ep.E; e++) cbm = std::max(cbm, p.cb[e]);
        const size_t smD = ((size_t)1 << cbm) * 4 + (size_t)X3_CAP * 8;
        cudaFuncSetAttribute(x3_chunksort, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smD);
        x3_chunksort<<<p.n_chunks, X3_T, smD, s>>>(p, ccnt, tmp2, pos, vals);
        count_launch();
        if (cudaGetLastError() != cudaSuccess) { st = cuda_fail(cudaGetLastError(), "index build sort"); break; }
    } while (0);
    cudaFreeAsync(scr, s);
    return st;
}

}  // namespace wmh
