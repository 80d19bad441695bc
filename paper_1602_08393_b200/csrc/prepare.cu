// prepare.cu -- a1 (column maxima), bound/structure validation, a3 (prefix sums,
// Eq. 3) and a4 (IntToComp, Alg. 4) on the device.
#include <stdarg.h>
#include <stdio.h>

#include <vector>

#include "common.cuh"

namespace wmh {

// ------------------------------------------------------------ a1: colmax
// Dense, 16-byte vectors: a 256-thread block owns a contiguous row range; its
// threads are (row phase g, column vector v) with V = D/16 vectors per row and
// G = 256 / V row phases, so consecutive threads read consecutive 16 B of a
// row (coalesced) and each thread keeps a per-byte running max (__vmaxu4)
// over rows g, g+G, ... with 4 loads in flight.  The G phases are merged in
// shared memory, then one atomicMax per nonzero column per block.  Reads
// N*D bytes once (HBM-bound).  Requires V <= 256.
__global__ void __launch_bounds__(256) colmax_dense_vec16(const uint8_t *__restrict__ x, int64_t n_rows,
                                                          int64_t dim, int64_t rows_per_block,
                                                          uint32_t *__restrict__ colmax) {
    __shared__ uint4 part[256];
    const int V = (int)(dim / 16), G = 256 / V;
    const int v = threadIdx.x % V, g = threadIdx.x / V;
    const int64_t r0 = (int64_t)blockIdx.x * rows_per_block;
    const int64_t r1 = min(n_rows, r0 + rows_per_block);
    uint4 acc = make_uint4(0, 0, 0, 0);
    if (g < G) {
        const uint4 *base = reinterpret_cast<const uint4 *>(x) + v;
        const int64_t stride = (int64_t)V;            // uint4s per row
        int64_t n = r0 + g;
        for (; n + 3 * G < r1; n += 4 * G) {
            const uint4 a = __ldg(base + n * stride), b = __ldg(base + (n + G) * stride);
            const uint4 c = __ldg(base + (n + 2 * G) * stride), d = __ldg(base + (n + 3 * G) * stride);
            acc.x = __vmaxu4(__vmaxu4(acc.x, a.x), __vmaxu4(__vmaxu4(b.x, c.x), d.x));
            acc.y = __vmaxu4(__vmaxu4(acc.y, a.y), __vmaxu4(__vmaxu4(b.y, c.y), d.y));
            acc.z = __vmaxu4(__vmaxu4(acc.z, a.z), __vmaxu4(__vmaxu4(b.z, c.z), d.z));
            acc.w = __vmaxu4(__vmaxu4(acc.w, a.w), __vmaxu4(__vmaxu4(b.w, c.w), d.w));
        }
        for (; n < r1; n += G) {
            const uint4 a = __ldg(base + n * stride);
            acc.x = __vmaxu4(acc.x, a.x); acc.y = __vmaxu4(acc.y, a.y);
            acc.z = __vmaxu4(acc.z, a.z); acc.w = __vmaxu4(acc.w, a.w);
        }
    }
    part[threadIdx.x] = acc;
    __syncthreads();
    if (g == 0) {
        for (int q = 1; q < G; q++) {
            const uint4 o = part[q * V + v];
            acc.x = __vmaxu4(acc.x, o.x); acc.y = __vmaxu4(acc.y, o.y);
            acc.z = __vmaxu4(acc.z, o.z); acc.w = __vmaxu4(acc.w, o.w);
        }
        const uint32_t w[4] = {acc.x, acc.y, acc.z, acc.w};
#pragma unroll
        for (int q = 0; q < 4; q++)
#pragma unroll
            for (int b = 0; b < 4; b++) {
                const uint32_t m = (w[q] >> (8 * b)) & 0xFFu;
                uint32_t *dst = &colmax[(int64_t)v * 16 + q * 4 + b];
                if (m > *((volatile uint32_t *)dst)) atomicMax(dst, m);   // skip when already reached
            }
    }
}

// Generic path (any dim / alignment / weight width).
template <typename W>
__global__ void colmax_dense_bytes(const W *__restrict__ x, int64_t n_rows, int64_t dim,
                                   int64_t rows_per_slice, uint32_t *__restrict__ colmax) {
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= dim) return;
    const int64_t r0 = (int64_t)blockIdx.y * rows_per_slice;
    const int64_t r1 = min(n_rows, r0 + rows_per_slice);
    uint32_t m = 0;
    for (int64_t n = r0; n < r1; n++) m = max(m, (uint32_t)x[n * dim + c]);
    if (m) atomicMax(&colmax[c], m);
}

// CSR: one thread per nonzero; read first, atomic only when it would raise the
// max (hot Zipf columns otherwise serialise on one address).
template <typename W>
__global__ void colmax_csr(const int32_t *__restrict__ col, const W *__restrict__ val, int64_t nnz,
                           uint32_t *__restrict__ colmax) {
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < nnz; e += (int64_t)gridDim.x * blockDim.x) {
        uint32_t v = val[e];
        int32_t c = col[e];
        if (v > *((volatile uint32_t *)&colmax[c])) atomicMax(&colmax[c], v);
    }
}

// ---------------------------------------------------------- validation
// First offending position, as a min-reduced 64-bit key.
template <typename W>
__global__ void check_dense_bounds(const W *__restrict__ x, int64_t n_rows, int64_t dim,
                                   const uint32_t *__restrict__ bounds, unsigned long long *first_bad) {
    for (int64_t n = blockIdx.x; n < n_rows; n += gridDim.x)
        for (int64_t c = threadIdx.x; c < dim; c += blockDim.x)
            if (x[n * dim + c] > bounds[c]) atomicMin(first_bad, (unsigned long long)(n * dim + c));
}

// Any column whose maximum exceeds its bound marks *bad (exact location later).
__global__ void colmax_exceeds(const uint32_t *__restrict__ cm, const uint32_t *__restrict__ bounds, int64_t dim,
                               unsigned long long *bad) {
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c < dim && cm[c] > bounds[c]) atomicMin(bad, (unsigned long long)c);
}

// One warp per row: row_ptr monotone, columns in range and strictly
// ascending, values within bounds.  key = (nnz index << 3) | code.
template <typename W>
__global__ void check_csr(const int64_t *__restrict__ row_ptr, const int32_t *__restrict__ col,
                          const W *__restrict__ val, int64_t n_rows, int64_t dim, int64_t nnz,
                          const uint32_t *__restrict__ bounds, unsigned long long *first_bad) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t n = warp; n < n_rows; n += nwarps) {
        int64_t a = row_ptr[n], b = row_ptr[n + 1];
        if (a > b || a < 0 || b > nnz || (n == 0 && a != 0) || (n == n_rows - 1 && b != nnz)) {
            if (lane == 0) atomicMin(first_bad, ((unsigned long long)(a < 0 ? 0 : a) << 3) | 4ull);
            continue;
        }
        for (int64_t e = a + lane; e < b; e += 32) {
            int32_t c = col[e];
            unsigned code = 0;
            if (c < 0 || c >= dim) code = 1;
            else if (e > a && col[e - 1] >= c) code = 2;
            else if (val[e] > bounds[c]) code = 3;
            if (code) atomicMin(first_bad, ((unsigned long long)e << 3) | code);
        }
    }
}

// Cells above 2^b - 1 in every column, b = 0..7: sum_c max(0, m_c - (2^b - 1)) --
// how many cells a tile whose planes clamp at b bits cannot test (the bit-plane
// tiles' clamp decision, read on the host without a device round trip)
__global__ void clamp_counts(const uint32_t *__restrict__ m, int64_t dim, unsigned long long *__restrict__ counts) {
    unsigned long long loc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < dim; c += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t v = m[c];
#pragma unroll
        for (int b = 0; b < 8; b++) loc[b] += v > (1u << b) - 1u ? v - ((1u << b) - 1u) : 0u;
    }
#pragma unroll
    for (int b = 0; b < 8; b++) {
        unsigned long long a = loc[b];
        for (int o = 16; o; o >>= 1) a += __shfl_xor_sync(0xFFFFFFFFu, a, o);
        if ((threadIdx.x & 31) == 0 && a) atomicAdd(counts + b, a);
    }
}

// ------------------------------------------------------- a3: prefix sums
constexpr int SCAN_B = 1024;

// Per-block sum, min and max of the bounds (u64 sums: overflow is detected, not wrapped).
__global__ void scan_block_sums(const uint32_t *__restrict__ m, int64_t dim, unsigned long long *__restrict__ sums,
                                unsigned int *__restrict__ mn, unsigned int *__restrict__ mx) {
    __shared__ unsigned long long ws[SCAN_B / 32];
    __shared__ unsigned int wmn[SCAN_B / 32], wmx[SCAN_B / 32];
    int64_t i = (int64_t)blockIdx.x * SCAN_B + threadIdx.x;
    uint32_t v = i < dim ? m[i] : 0u;
    unsigned long long s = v;
    unsigned int lo = i < dim ? v : 0xFFFFFFFFu, hi = v;
    for (int o = 16; o; o >>= 1) {
        s += __shfl_xor_sync(0xFFFFFFFFu, s, o);
        lo = min(lo, __shfl_xor_sync(0xFFFFFFFFu, lo, o));
        hi = max(hi, __shfl_xor_sync(0xFFFFFFFFu, hi, o));
    }
    if ((threadIdx.x & 31) == 0) { ws[threadIdx.x >> 5] = s; wmn[threadIdx.x >> 5] = lo; wmx[threadIdx.x >> 5] = hi; }
    __syncthreads();
    if (threadIdx.x < 32) {
        s = ws[threadIdx.x];
        lo = wmn[threadIdx.x];
        hi = wmx[threadIdx.x];
        for (int o = 16; o; o >>= 1) {
            s += __shfl_xor_sync(0xFFFFFFFFu, s, o);
            lo = min(lo, __shfl_xor_sync(0xFFFFFFFFu, lo, o));
            hi = max(hi, __shfl_xor_sync(0xFFFFFFFFu, hi, o));
        }
        if (threadIdx.x == 0) { sums[blockIdx.x] = s; atomicMin(mn, lo); atomicMax(mx, hi); }
    }
}

// Exclusive scan of the block sums in one block (looping over 1024-wide
// segments); writes total M to *M_out.
__global__ void scan_sums_single(unsigned long long *__restrict__ sums, int64_t nblocks,
                                 unsigned long long *__restrict__ M_out) {
    __shared__ unsigned long long wtot[SCAN_B / 32];
    __shared__ unsigned long long carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (int64_t base = 0; base < nblocks; base += SCAN_B) {
        int64_t i = base + threadIdx.x;
        unsigned long long v = i < nblocks ? sums[i] : 0ull;
        unsigned long long inc = v;                       // warp inclusive scan
        for (int o = 1; o < 32; o <<= 1) {
            unsigned long long t = __shfl_up_sync(0xFFFFFFFFu, inc, o);
            if ((threadIdx.x & 31) >= o) inc += t;
        }
        if ((threadIdx.x & 31) == 31) wtot[threadIdx.x >> 5] = inc;
        __syncthreads();
        if (threadIdx.x < 32) {
            unsigned long long w = wtot[threadIdx.x], wi = w;
            for (int o = 1; o < 32; o <<= 1) {
                unsigned long long t = __shfl_up_sync(0xFFFFFFFFu, wi, o);
                if (threadIdx.x >= o) wi += t;
            }
            wtot[threadIdx.x] = wi - w;                   // exclusive warp offsets
        }
        __syncthreads();
        unsigned long long excl = carry + wtot[threadIdx.x >> 5] + inc - v;
        if (i < nblocks) sums[i] = excl;
        __syncthreads();
        if (threadIdx.x == SCAN_B - 1) carry = excl + v;
        __syncthreads();
    }
    if (threadIdx.x == 0) *M_out = carry;
}

// comp_to_m[c] = sums[block] + exclusive in-block prefix (as u32; the host
// rejects M >= 2^32 before any table is used).  comp_to_m[dim] = M.
__global__ void scan_apply(const uint32_t *__restrict__ m, int64_t dim, const unsigned long long *__restrict__ sums,
                          const unsigned long long *__restrict__ M_total, uint32_t *__restrict__ comp_to_m) {
    __shared__ unsigned long long wtot[SCAN_B / 32];
    int64_t i = (int64_t)blockIdx.x * SCAN_B + threadIdx.x;
    unsigned long long v = i < dim ? m[i] : 0u;
    unsigned long long inc = v;
    for (int o = 1; o < 32; o <<= 1) {
        unsigned long long t = __shfl_up_sync(0xFFFFFFFFu, inc, o);
        if ((threadIdx.x & 31) >= o) inc += t;
    }
    if ((threadIdx.x & 31) == 31) wtot[threadIdx.x >> 5] = inc;
    __syncthreads();
    if (threadIdx.x < 32) {
        unsigned long long w = wtot[threadIdx.x], wi = w;
        for (int o = 1; o < 32; o <<= 1) {
            unsigned long long t = __shfl_up_sync(0xFFFFFFFFu, wi, o);
            if (threadIdx.x >= o) wi += t;
        }
        wtot[threadIdx.x] = wi - w;
    }
    __syncthreads();
    if (i < dim) comp_to_m[i] = (uint32_t)(sums[blockIdx.x] + wtot[threadIdx.x >> 5] + inc - v);
    if (i == 0) comp_to_m[dim] = (uint32_t)(*M_total);
}

// ----------------------------------------------------------- a4: IntToComp
// One warp per component c: lanes write IntToComp[t] = c and the packed
// form (c << 8) | (t - CompToM[c]) for t in [CompToM[c], CompToM[c+1]).
// Zero-width components write nothing (reading R11).
__global__ void fill_int_to_comp(const uint32_t *__restrict__ comp_to_m, int64_t dim, uint32_t *__restrict__ i2c,
                                 uint32_t *__restrict__ pack) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t c = warp; c < dim; c += nwarps) {
        uint32_t a = comp_to_m[c], b = comp_to_m[c + 1];
        for (uint32_t t = a + lane; t < b; t += 32) {
            i2c[t] = (uint32_t)c;
            if (pack) pack[t] = ((uint32_t)c << 8) | (t - a);
        }
    }
}

}  // namespace wmh

using namespace wmh;

// ===================================================================== C ABI
// ------------------------------------------------ row-sum statistics
// hist[b] += 1 for a row with |x|_1 in [2^b, 2^(b+1)); hist[64] counts empty
// rows.  Warp per row.  The index kernel sizes its draw horizon from the
// 0.1% quantile (Theorem 2: a row needs ~1/s draws, s = |x|_1 / M, Eq. 17).
template <typename W>
__global__ void __launch_bounds__(256) rowsum_hist(const W *__restrict__ dense, const int64_t *__restrict__ row_ptr,
                                                   const W *__restrict__ val, int64_t n_rows, int64_t dim,
                                                   unsigned long long *__restrict__ hist) {
    const int lane = threadIdx.x & 31;
    const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    unsigned long long total = 0;                 // hist[65]: sum of all row sums
    uint32_t ge[8] = {0, 0, 0, 0, 0, 0, 0, 0};   // hist[66 + b]: sampled weights >= 2^b - 1 (b = 3..7), hist[74]: cells sampled
    uint32_t cells = 0;
    for (int64_t r = w0; r < n_rows; r += nw) {
        unsigned long long s = 0;
        if (dense) {
            const W *x = dense + r * dim;
            if (sizeof(W) == 1 && (dim & 3) == 0 && ((uintptr_t)dense & 3) == 0) {
                const uint32_t *x4 = reinterpret_cast<const uint32_t *>(x);
                const bool sample = (r & 15) == 0;   // every 16th row: the value tail the bit-sliced tile clamps
                for (int64_t i = lane; i < dim / 4; i += 32) {
                    const uint32_t v = __ldg(x4 + i);
                    s += __dp4a(v, 0x01010101u, 0u);
                    if (sample) {
#pragma unroll
                        for (int b = 3; b < 8; b++) ge[b] += __popc(__vcmpgeu4(v, ((1u << b) - 1u) * 0x01010101u)) >> 3;
                        cells += 4;
                    }
                }
            } else {
                for (int64_t i = lane; i < dim; i += 32) s += __ldg(x + i);
            }
        } else {
            const int64_t a = row_ptr[r], b = row_ptr[r + 1];
            for (int64_t i = a + lane; i < b; i += 32) s += __ldg(val + i);
        }
        for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xFFFFFFFFu, s, o);
        if (lane == 0) atomicAdd(hist + (s ? 63 - __clzll((long long)s) : 64), 1ull);
        total += s;
    }
    if (lane == 0 && total) atomicAdd(hist + 65, total);
#pragma unroll
    for (int b = 3; b < 8; b++) {
        uint32_t a = ge[b];
        for (int o = 16; o; o >>= 1) a += __shfl_xor_sync(0xFFFFFFFFu, a, o);
        if (lane == 0 && a) atomicAdd(hist + 66 + b, (unsigned long long)a);
    }
    for (int o = 16; o; o >>= 1) cells += __shfl_xor_sync(0xFFFFFFFFu, cells, o);
    if (lane == 0 && cells) atomicAdd(hist + 74, (unsigned long long)cells);
}

extern "C" wmh_status wmh_colmax(const wmh_rows *rows, uint32_t *colmax, void *stream) {
    wmh_status st = check_rows(rows, true);
    if (st != WMH_OK) return st;
    if (!colmax) { set_error("wmh_colmax: colmax is NULL"); return WMH_EINVAL; }
    cudaStream_t s = (cudaStream_t)stream;
    WMH_CUDA_TRY(cudaMemsetAsync(colmax, 0, sizeof(uint32_t) * rows->dim, s), "memset colmax");
    if (rows->n_rows == 0) return WMH_OK;
    const bool w16 = weight_bytes(*rows) == 2;
    const uint16_t *dense16 = reinterpret_cast<const uint16_t *>(rows->dense);
    const uint16_t *val16 = reinterpret_cast<const uint16_t *>(rows->val);
    if (rows->kind == WMH_DENSE) {
        const int sms = num_sms();
        const bool vec = !w16 && (rows->dim % 16 == 0) && (rows->dim / 16 <= 256) && ((uintptr_t)rows->dense % 16 == 0);
        if (vec) {
            const int64_t blocks = min(rows->n_rows, (int64_t)sms * 4);
            const int64_t per = (rows->n_rows + blocks - 1) / blocks;
            colmax_dense_vec16<<<(unsigned)((rows->n_rows + per - 1) / per), 256, 0, s>>>(rows->dense, rows->n_rows,
                                                                                     rows->dim, per, colmax);
        } else {
            const int threads = 128;
            const int64_t gx = (rows->dim + threads - 1) / threads;
            int64_t gy = max((int64_t)1, min(rows->n_rows, (int64_t)sms * 8 / max((int64_t)1, gx)));
            gy = min(gy, (int64_t)65535);
            const int64_t per = (rows->n_rows + gy - 1) / gy;
            gy = (rows->n_rows + per - 1) / per;
            if (w16)
                colmax_dense_bytes<<<dim3((unsigned)gx, (unsigned)gy), threads, 0, s>>>(dense16, rows->n_rows,
                                                                                      rows->dim, per, colmax);
            else
                colmax_dense_bytes<<<dim3((unsigned)gx, (unsigned)gy), threads, 0, s>>>(rows->dense, rows->n_rows,
                                                                                      rows->dim, per, colmax);
        }
    } else {
        if (rows->nnz > 0) {
            int64_t blocks = min((int64_t)num_sms() * 16, (rows->nnz + 255) / 256);
            if (w16) colmax_csr<<<(unsigned)blocks, 256, 0, s>>>(rows->col, val16, rows->nnz, colmax);
            else colmax_csr<<<(unsigned)blocks, 256, 0, s>>>(rows->col, rows->val, rows->nnz, colmax);
        }
    }
    WMH_LAUNCH_CHECK("colmax launch");
    return WMH_OK;
}

extern "C" wmh_status wmh_prepare(const uint32_t *bounds, int64_t dim, const wmh_rows *rows, wmh_layout **out,
                                  void *stream) {
    if (!out) { set_error("wmh_prepare: out is NULL"); return WMH_EINVAL; }
    *out = nullptr;
    if (!bounds) { set_error("wmh_prepare: bounds is NULL"); return WMH_EINVAL; }
    if (dim < 1 || dim > (1ll << 24)) { set_error("wmh_prepare: dim=%lld outside [1, 2^24]", (long long)dim); return WMH_EINVAL; }
    if (rows) {
        wmh_status st = check_rows(rows, true);
        if (st != WMH_OK) return st;
        if (rows->dim != dim) { set_error("wmh_prepare: rows->dim=%lld != dim=%lld", (long long)rows->dim, (long long)dim); return WMH_EINVAL; }
    }
    cudaStream_t s = (cudaStream_t)stream;
    int dev = 0;
    WMH_CUDA_TRY(cudaGetDevice(&dev), "cudaGetDevice");

    wmh_layout *L = new wmh_layout();
    L->dim = dim;
    L->device = dev;
    auto fail = [&](wmh_status st) { wmh_layout_free(L); return st; };

    if (cudaMalloc(&L->bounds, sizeof(uint32_t) * dim) != cudaSuccess ||
        cudaMalloc(&L->comp_to_m, sizeof(uint32_t) * (dim + 1)) != cudaSuccess) {
        set_error("wmh_prepare: cudaMalloc of %lld-entry tables failed", (long long)dim);
        return fail(WMH_ENOMEM);
    }
    if (cudaMemcpyAsync(L->bounds, bounds, sizeof(uint32_t) * dim, cudaMemcpyDeviceToDevice, s) != cudaSuccess)
        return fail(cuda_fail(cudaGetLastError(), "copy bounds"));

    const int64_t nb = (dim + SCAN_B - 1) / SCAN_B;
    // scratch: sums[nb], M, first_bad, mn, mx, pad, the 8 clamp counts, colmax[dim] (dense validation)
    unsigned long long *scr = nullptr;
    size_t scr_bytes = sizeof(unsigned long long) * (nb + 12) + sizeof(uint32_t) * dim;
    if (cudaMallocAsync((void **)&scr, scr_bytes, s) != cudaSuccess) {
        set_error("wmh_prepare: scratch alloc failed");
        return fail(WMH_ENOMEM);
    }
    unsigned long long *sums = scr, *Mdev = scr + nb, *bad = scr + nb + 1;
    unsigned int *mnmx = reinterpret_cast<unsigned int *>(scr + nb + 2);
    unsigned long long init[12] = {0ull, ~0ull, 0x00000000FFFFFFFFull, 0ull};  // M, bad, {mn=~0,mx=0}, pad, counts
    cudaMemcpyAsync(Mdev, init, sizeof(init), cudaMemcpyHostToDevice, s);

    const int sms = num_sms();
    if (rows && rows->n_rows > 0) {
        if (rows->kind == WMH_DENSE) {
            // fast path: column maxima (one HBM pass) against the bounds; the
            // exact first offender is located only when a column fails
            uint32_t *cm = reinterpret_cast<uint32_t *>(scr + nb + 12);
            wmh_status cst = wmh_colmax(rows, cm, stream);
            if (cst != WMH_OK) { cudaFreeAsync(scr, s); return fail(cst); }
            colmax_exceeds<<<(unsigned)((dim + 255) / 256), 256, 0, s>>>(cm, L->bounds, dim, bad);
        } else
        {
            if (weight_bytes(*rows) == 2)
                check_csr<<<sms * 8, 256, 0, s>>>(rows->row_ptr, rows->col, reinterpret_cast<const uint16_t *>(rows->val),
                                                  rows->n_rows, dim, rows->nnz, L->bounds, bad);
            else
                check_csr<<<sms * 8, 256, 0, s>>>(rows->row_ptr, rows->col, rows->val, rows->n_rows, dim, rows->nnz,
                                                  L->bounds, bad);
        }
    }
    unsigned long long *hist = nullptr, hhist[75] = {0};
    const bool stats = rows && rows->n_rows > 0;
    if (stats) {
        if (cudaMallocAsync((void **)&hist, sizeof hhist, s) != cudaSuccess) { cudaFreeAsync(scr, s); set_error("wmh_prepare: scratch alloc failed"); return fail(WMH_ENOMEM); }
        cudaMemsetAsync(hist, 0, sizeof hhist, s);
        if (weight_bytes(*rows) == 2)
            rowsum_hist<<<sms * 8, 256, 0, s>>>(rows->kind == WMH_DENSE ? reinterpret_cast<const uint16_t *>(rows->dense) : nullptr,
                                                rows->row_ptr, reinterpret_cast<const uint16_t *>(rows->val), rows->n_rows, dim, hist);
        else
            rowsum_hist<<<sms * 8, 256, 0, s>>>(rows->kind == WMH_DENSE ? rows->dense : nullptr, rows->row_ptr, rows->val,
                                                rows->n_rows, dim, hist);
        count_launch();
        cudaMemcpyAsync(hhist, hist, sizeof hhist, cudaMemcpyDeviceToHost, s);
    }
    scan_block_sums<<<(unsigned)nb, SCAN_B, 0, s>>>(L->bounds, dim, sums, mnmx, mnmx + 1);
    scan_sums_single<<<1, SCAN_B, 0, s>>>(sums, nb, Mdev);
    scan_apply<<<(unsigned)nb, SCAN_B, 0, s>>>(L->bounds, dim, sums, Mdev, L->comp_to_m);
    clamp_counts<<<(unsigned)std::min<int64_t>(sms * 4, (dim + 255) / 256), 256, 0, s>>>(L->bounds, dim, Mdev + 4);
    count_launch(4 + ((rows && rows->n_rows > 0) ? 1 : 0));
    if (cudaGetLastError() != cudaSuccess) { cudaFreeAsync(scr, s); return fail(cuda_fail(cudaGetLastError(), "prepare scan launch")); }

    unsigned long long host[12];
    cudaError_t e1 = cudaMemcpyAsync(host, Mdev, sizeof(host), cudaMemcpyDeviceToHost, s);
    cudaError_t e2 = cudaStreamSynchronize(s);
    cudaFreeAsync(scr, s);
    if (hist) cudaFreeAsync(hist, s);
    if (e1 != cudaSuccess || e2 != cudaSuccess) return fail(cuda_fail(e1 != cudaSuccess ? e1 : e2, "prepare readback"));
    if (stats) {
        for (int b = 0; b < 8; b++) L->value_ge[b] = hhist[66 + b];
        L->value_cells = hhist[74];
    }
    if (stats) {             // 0.1% quantile of the nonzero row sums, as the bin's lower end 2^b; mean s
        L->mean_s = host[0] ? (double)hhist[65] / ((double)rows->n_rows * (double)host[0]) : -1.0;
        unsigned long long nz = 0, run = 0;
        for (int b = 0; b < 64; b++) nz += hhist[b];
        for (int b = 0; b < 64 && nz; b++) {
            run += hhist[b];
            if (run * 1000 > nz) { L->rowsum_q = 1ull << b; break; }
        }
    }
    const unsigned long long M = host[0], first_bad = host[1];
    const unsigned int mn = (unsigned int)(host[2] & 0xFFFFFFFFu), mx = (unsigned int)(host[2] >> 32);

    if (mx > 65535) { set_error("wmh_prepare: a bound is %u > 65535 (weights are at most uint16)", mx); return fail(WMH_EINVAL); }
    if (first_bad != ~0ull) {
        if (rows->kind == WMH_DENSE) {
            // slow path: locate the first offending (row, col)
            unsigned long long *b2 = nullptr, fb = ~0ull;
            if (cudaMallocAsync((void **)&b2, sizeof fb, s) != cudaSuccess) return fail(WMH_ENOMEM);
            cudaMemcpyAsync(b2, &fb, sizeof fb, cudaMemcpyHostToDevice, s);
            if (weight_bytes(*rows) == 2)
                check_dense_bounds<<<sms * 8, 256, 0, s>>>(reinterpret_cast<const uint16_t *>(rows->dense), rows->n_rows, dim,
                                                           L->bounds, b2);
            else
                check_dense_bounds<<<sms * 8, 256, 0, s>>>(rows->dense, rows->n_rows, dim, L->bounds, b2);
            count_launch();
            cudaMemcpyAsync(&fb, b2, sizeof fb, cudaMemcpyDeviceToHost, s);
            cudaError_t e3 = cudaStreamSynchronize(s);
            cudaFreeAsync(b2, s);
            if (e3 != cudaSuccess) return fail(cuda_fail(e3, "prepare bound check"));
            long long r = (long long)(fb / (unsigned long long)dim), c = (long long)(fb % (unsigned long long)dim);
            set_error("wmh_prepare: weight x[%lld][%lld] exceeds its bound", r, c);
            return fail(WMH_EBOUND);
        }
        unsigned code = (unsigned)(first_bad & 7ull);
        long long e = (long long)(first_bad >> 3);
        static const char *what[] = {"", "column index out of range", "columns not strictly ascending",
                                     "value exceeds its bound", "row_ptr malformed"};
        set_error("wmh_prepare: CSR nonzero %lld: %s", e, what[code <= 4 ? code : 0]);
        return fail(code == 3 ? WMH_EBOUND : WMH_EINVAL);
    }
    if (M == 0) { set_error("wmh_prepare: M = sum of bounds is 0"); return fail(WMH_EEMPTY); }
    if (M >= (1ull << 32)) { set_error("wmh_prepare: M = %llu >= 2^32", M); return fail(WMH_EOVERFLOW); }
    L->M = M;
    if (mn == mx) { L->flags |= WMH_LAYOUT_UNIFORM; L->uniform_m = mx; }
    L->max_bound = (uint32_t)mx;
    for (int b = 0; b < 8; b++) L->clamp_cells[b] = host[4 + b];
    if (mx > 255) L->flags |= WMH_LAYOUT_WIDE;       // 8-bit cell offsets no longer fit: no cell_pack

    if (cudaMalloc(&L->int_to_comp, sizeof(uint32_t) * M) != cudaSuccess ||
        (!(L->flags & WMH_LAYOUT_WIDE) && cudaMalloc(&L->cell_pack, sizeof(uint32_t) * M) != cudaSuccess)) {
        set_error("wmh_prepare: cudaMalloc of IntToComp (%llu cells) failed", M);
        return fail(WMH_ENOMEM);
    }
    int64_t blocks = min((int64_t)sms * 16, (dim * 32 + 255) / 256);
    fill_int_to_comp<<<(unsigned)blocks, 256, 0, s>>>(L->comp_to_m, dim, L->int_to_comp, L->cell_pack);
    count_launch();
    if (cudaGetLastError() != cudaSuccess) return fail(cuda_fail(cudaGetLastError(), "fill IntToComp launch"));
    {   // layout digest: FNV-1a (64-bit) over dim and the bounds, for "same layout" checks
        std::vector<uint32_t> hb((size_t)dim);
        cudaError_t e1 = cudaMemcpyAsync(hb.data(), L->bounds, sizeof(uint32_t) * dim, cudaMemcpyDeviceToHost, s);
        cudaError_t e2 = cudaStreamSynchronize(s);
        if (e1 != cudaSuccess || e2 != cudaSuccess) return fail(cuda_fail(e1 != cudaSuccess ? e1 : e2, "layout digest"));
        uint64_t h = 0xcbf29ce484222325ull;
        auto mix = [&](uint64_t v) {
            for (int i = 0; i < 8; i++) { h ^= (v >> (8 * i)) & 0xFFu; h *= 0x100000001b3ull; }
        };
        mix((uint64_t)dim);
        for (uint32_t b : hb) mix(b);
        L->digest = h;
    }
    *out = L;
    return WMH_OK;
}

// Rows against an existing layout (Eq. 2 needs x_c <= m_c for every row that is
// hashed, not only for the rows prepare saw): the same checks as wmh_prepare's
// bounds pass -- one column-max pass for dense rows (the first offender located
// only when a column fails), one warp per CSR row.  Synchronises once.
extern "C" wmh_status wmh_check_rows(const wmh_layout *L, const wmh_rows *rows, void *stream) {
    if (!L) { set_error("wmh_check_rows: layout is NULL"); return WMH_EINVAL; }
    wmh_status st = check_rows(rows, true);
    if (st != WMH_OK) return st;
    if (rows->dim != L->dim) { set_error("wmh_check_rows: rows dim %lld != layout dim %lld", (long long)rows->dim, (long long)L->dim); return WMH_EINVAL; }
    if (rows->n_rows == 0) return WMH_OK;
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t dim = L->dim;
    const int sms = num_sms();
    uint8_t *scr = nullptr;
    const size_t scr_b = 256 + (rows->kind == WMH_DENSE ? sizeof(uint32_t) * (size_t)dim : 0);
    WMH_CUDA_TRY(cudaMallocAsync((void **)&scr, scr_b, s), "check_rows scratch alloc");
    unsigned long long *bad = reinterpret_cast<unsigned long long *>(scr);
    unsigned long long fb = ~0ull;
    cudaMemcpyAsync(bad, &fb, sizeof fb, cudaMemcpyHostToDevice, s);
    if (rows->kind == WMH_DENSE) {
        uint32_t *cm = reinterpret_cast<uint32_t *>(scr + 256);
        st = wmh_colmax(rows, cm, stream);
        if (st != WMH_OK) { cudaFreeAsync(scr, s); return st; }
        colmax_exceeds<<<(unsigned)((dim + 255) / 256), 256, 0, s>>>(cm, L->bounds, dim, bad);
    } else if (weight_bytes(*rows) == 2) {
        check_csr<<<sms * 8, 256, 0, s>>>(rows->row_ptr, rows->col, reinterpret_cast<const uint16_t *>(rows->val),
                                          rows->n_rows, dim, rows->nnz, L->bounds, bad);
    } else {
        check_csr<<<sms * 8, 256, 0, s>>>(rows->row_ptr, rows->col, rows->val, rows->n_rows, dim, rows->nnz, L->bounds, bad);
    }
    count_launch();
    cudaMemcpyAsync(&fb, bad, sizeof fb, cudaMemcpyDeviceToHost, s);
    cudaError_t e = cudaStreamSynchronize(s);
    if (e == cudaSuccess && fb != ~0ull && rows->kind == WMH_DENSE) {      // locate the first offender
        fb = ~0ull;
        cudaMemcpyAsync(bad, &fb, sizeof fb, cudaMemcpyHostToDevice, s);
        if (weight_bytes(*rows) == 2)
            check_dense_bounds<<<sms * 8, 256, 0, s>>>(reinterpret_cast<const uint16_t *>(rows->dense), rows->n_rows, dim,
                                                       L->bounds, bad);
        else
            check_dense_bounds<<<sms * 8, 256, 0, s>>>(rows->dense, rows->n_rows, dim, L->bounds, bad);
        count_launch();
        cudaMemcpyAsync(&fb, bad, sizeof fb, cudaMemcpyDeviceToHost, s);
        e = cudaStreamSynchronize(s);
        if (e == cudaSuccess) {
            cudaFreeAsync(scr, s);
            set_error("wmh_check_rows: weight x[%lld][%lld] exceeds its bound", (long long)(fb / (unsigned long long)dim),
                      (long long)(fb % (unsigned long long)dim));
            return WMH_EBOUND;
        }
    }
    cudaFreeAsync(scr, s);
    if (e != cudaSuccess) return cuda_fail(e, "check_rows readback");
    if (fb != ~0ull) {
        const unsigned code = (unsigned)(fb & 7ull);
        static const char *what[] = {"", "column index out of range", "columns not strictly ascending",
                                     "value exceeds its bound", "row_ptr malformed"};
        set_error("wmh_check_rows: CSR nonzero %lld: %s", (long long)(fb >> 3), what[code <= 4 ? code : 0]);
        return code == 3 ? WMH_EBOUND : WMH_EINVAL;
    }
    return WMH_OK;
}

extern "C" wmh_status wmh_layout_digest(const wmh_layout *L, uint64_t *digest) {
    if (!L || !digest) { set_error("wmh_layout_digest: NULL argument"); return WMH_EINVAL; }
    *digest = L->digest;
    return WMH_OK;
}

extern "C" wmh_status wmh_layout_info(const wmh_layout *L, int64_t *dim, uint64_t *M, uint32_t *flags,
                                      uint32_t *uniform_bound) {
    if (!L) { set_error("wmh_layout_info: layout is NULL"); return WMH_EINVAL; }
    if (dim) *dim = L->dim;
    if (M) *M = L->M;
    if (flags) *flags = L->flags;
    if (uniform_bound) *uniform_bound = L->uniform_m;
    return WMH_OK;
}

extern "C" wmh_status wmh_layout_tables(const wmh_layout *L, const uint32_t **c2m, const uint32_t **i2c,
                                        const uint32_t **bounds) {
    if (!L) { set_error("wmh_layout_tables: layout is NULL"); return WMH_EINVAL; }
    if (c2m) *c2m = L->comp_to_m;
    if (i2c) *i2c = L->int_to_comp;
    if (bounds) *bounds = L->bounds;
    return WMH_OK;
}

extern "C" void wmh_layout_free(wmh_layout *L) {
    if (!L) return;
    cudaFree(L->bounds);
    cudaFree(L->comp_to_m);
    cudaFree(L->int_to_comp);
    cudaFree(L->cell_pack);
    delete L;
}
