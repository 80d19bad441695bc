// hash_simple.cu -- WMH_ALGO_SIMPLE: the paper's procedure mapped one thread per
// (row, hash j), every step through global tables.  Kept as the measured
// baseline for the tiled kernel and as the path for shapes the tiled kernel
// does not take.
//
// Per thread: Alg. 3's while loop over the counter stream
// r_t (common.cuh), Alg. 5's ISGREEN with IntToComp/CompToM fused
// into one packed load cell_pack[r] = (c << 8) | (r - CompToM[c]) (exact since
// every bound <= 255; wide layouts use the two lookups), and the saturating cap
// (reading R9).  Weights uint8 or uint16 (fixed-point real data).
#include "common.cuh"

namespace wmh {

// x_c of a CSR row by binary search over its ascending columns (Sec. 3.3's
// O(log d) search, applied to the row's support).
template <typename W>
__device__ __forceinline__ uint32_t csr_value(const int32_t *__restrict__ col, const W *__restrict__ val,
                                              int64_t a, int64_t b, uint32_t c) {
    int64_t lo = a, hi = b;                       // first index with col >= c
    while (lo < hi) {
        int64_t mid = (lo + hi) >> 1;
        if ((uint32_t)__ldg(col + mid) < c) lo = mid + 1;
        else hi = mid;
    }
    return (lo < b && (uint32_t)__ldg(col + lo) == c) ? (uint32_t)__ldg(val + lo) : 0u;
}

template <int SIGB, bool CSR, typename W, bool BSEARCH = false>
__global__ void __launch_bounds__(256) hash_simple_kernel(
    const W *__restrict__ dense, const int64_t *__restrict__ row_ptr, const int32_t *__restrict__ col,
    const W *__restrict__ val, int64_t n_rows, int64_t dim, const uint32_t *__restrict__ pack, uint32_t uni_m,
    const uint32_t *__restrict__ i2c, const uint32_t *__restrict__ c2m, uint32_t M,
    uint64_t S, uint32_t k, uint32_t cap, void *__restrict__ sig, unsigned long long *__restrict__ n_sat) {
    const int64_t total = n_rows * (int64_t)k;
    unsigned int sat = 0;
    for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int64_t n = idx / k;
        const uint32_t j = (uint32_t)(idx - n * (int64_t)k);
        const uint64_t keyj = S ^ ((uint64_t)j << 32);
        int64_t a = 0, b = 0;
        if (CSR) { a = __ldg(row_ptr + n); b = __ldg(row_ptr + n + 1); }
        uint32_t h = cap;
        bool found = false;
        if (!CSR || a < b) {
            for (uint32_t t = 0; t < cap; t++) {
                const uint32_t r = mulhi_range(splitmix64(keyj ^ (uint64_t)t), M);
                const uint2 cell = BSEARCH ? cell_bsearch(r, c2m, (uint32_t)dim) : cell_lookup(r, pack, uni_m, i2c, c2m);
                const uint32_t c = cell.x, off = cell.y;
                uint32_t xv;
                if (CSR) xv = csr_value(col, val, a, b, c);
                else xv = __ldg(dense + n * dim + c);
                if (off < xv) { h = t + 1; found = true; break; }
            }
        }
        sat += !found;
        if (SIGB == 1) reinterpret_cast<uint8_t *>(sig)[idx] = (uint8_t)h;
        else reinterpret_cast<uint16_t *>(sig)[idx] = (uint16_t)h;
    }
    if (n_sat) {
        for (int o = 16; o; o >>= 1) sat += __shfl_xor_sync(0xFFFFFFFFu, sat, o);
        if ((threadIdx.x & 31) == 0 && sat) atomicAdd(n_sat, (unsigned long long)sat);
    }
}

wmh_status launch_hash_simple(const HashArgs &a) {
    const int64_t total = a.rows.n_rows * (int64_t)a.k;
    if (total == 0) return WMH_OK;
    const int threads = 256;
    int64_t blocks = min((int64_t)num_sms() * 32, (total + threads - 1) / threads);
    const uint32_t M = (uint32_t)a.L->M;
    const bool csr = a.rows.kind == WMH_CSR;
    const uint32_t uni_m = (a.L->flags & WMH_LAYOUT_UNIFORM) ? a.L->uniform_m : 0u;
    const uint32_t *pack = (a.L->flags & WMH_LAYOUT_WIDE) ? nullptr : a.L->cell_pack;
#define WMH_SIMPLE(SB, CS, W)                                                                                    \
    (a.isgreen_bsearch ? hash_simple_kernel<SB, CS, W, true> : hash_simple_kernel<SB, CS, W, false>)             \
        <<<(unsigned)blocks, threads, 0, a.stream>>>(                                                            \
        reinterpret_cast<const W *>(a.rows.dense), a.rows.row_ptr, a.rows.col, reinterpret_cast<const W *>(a.rows.val), \
        a.rows.n_rows, a.rows.dim, pack, uni_m, a.L->int_to_comp, a.L->comp_to_m, M, a.S, a.k, a.cap, a.sig, a.n_sat)
    kernel_timer_begin(a.stream);
    if (weight_bytes(a.rows) == 2) {
        if (a.sig_bytes == 1) { if (csr) WMH_SIMPLE(1, true, uint16_t); else WMH_SIMPLE(1, false, uint16_t); }
        else { if (csr) WMH_SIMPLE(2, true, uint16_t); else WMH_SIMPLE(2, false, uint16_t); }
    } else {
        if (a.sig_bytes == 1) { if (csr) WMH_SIMPLE(1, true, uint8_t); else WMH_SIMPLE(1, false, uint8_t); }
        else { if (csr) WMH_SIMPLE(2, true, uint8_t); else WMH_SIMPLE(2, false, uint8_t); }
    }
    kernel_timer_end(a.stream);
#undef WMH_SIMPLE
    WMH_LAUNCH_CHECK("hash_simple launch");
    return WMH_OK;
}

}  // namespace wmh
