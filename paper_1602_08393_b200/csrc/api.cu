// api.cu -- the C ABI (include/wmh.h): argument validation, hash dispatch, the
// host-buffer e2e entry, collide (a10, Eq. 14-15) and error reporting.
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include <mutex>
#include <vector>

#include "common.cuh"

namespace wmh {

static thread_local char g_err[512] = "";

void set_error(const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
}

wmh_status cuda_fail(cudaError_t e, const char *what) {
    set_error("%s: CUDA error %d (%s)", what, (int)e, cudaGetErrorString(e));
    return e == cudaErrorMemoryAllocation ? WMH_ENOMEM : WMH_ECUDA;
}

int num_sms() {
    static int cached[64] = {0};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
    if (!cached[dev]) {
        int v = 0;
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        cached[dev] = v > 0 ? v : 148;
    }
    return cached[dev];
}

wmh_status check_rows(const wmh_rows *rows, bool need_data) {
    if (!rows) { set_error("rows is NULL"); return WMH_EINVAL; }
    if (rows->n_rows < 0) { set_error("n_rows=%lld < 0", (long long)rows->n_rows); return WMH_EINVAL; }
    if (rows->dim < 1) { set_error("dim=%lld < 1", (long long)rows->dim); return WMH_EINVAL; }
    if (rows->kind == WMH_DENSE) {
        if (need_data && rows->n_rows > 0 && !rows->dense) { set_error("dense rows pointer is NULL"); return WMH_EINVAL; }
    } else if (rows->kind == WMH_CSR) {
        if (rows->nnz < 0) { set_error("nnz=%lld < 0", (long long)rows->nnz); return WMH_EINVAL; }
        if (need_data && rows->n_rows > 0 && !rows->row_ptr) { set_error("CSR row_ptr is NULL"); return WMH_EINVAL; }
        if (need_data && rows->nnz > 0 && (!rows->col || !rows->val)) { set_error("CSR col/val is NULL"); return WMH_EINVAL; }
        if (rows->nnz >= (1ll << 40)) { set_error("nnz too large"); return WMH_EINVAL; }
    } else {
        set_error("unknown rows kind %d", (int)rows->kind);
        return WMH_EINVAL;
    }
    return WMH_OK;
}

// ------------------------------------------------------------- a10 collide
// One warp per pair; 16-byte vector loads when the signature rows are
// 16-byte aligned, a scalar lane-strided loop otherwise.  Equal halves /
// bytes are counted from the xor of the two words.
template <int SIGB, bool VEC>
__global__ void __launch_bounds__(256) collide_kernel(const uint8_t *__restrict__ sig, uint32_t k, int64_t n_rows,
                                                      const int64_t *__restrict__ pairs, int64_t n_pairs,
                                                      uint32_t *__restrict__ matches, float *__restrict__ jhat,
                                                      unsigned long long *__restrict__ n_bad) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int64_t row_bytes = (int64_t)k * SIGB;
    for (int64_t p = warp; p < n_pairs; p += nwarps) {
        const int64_t a = __ldg(pairs + 2 * p), b = __ldg(pairs + 2 * p + 1);
        if (a < 0 || b < 0 || a >= n_rows || b >= n_rows) {
            if (lane == 0) {
                matches[p] = 0;
                if (jhat) jhat[p] = __int_as_float(0x7fc00000);
                if (n_bad) atomicAdd(n_bad, 1ull);
            }
            continue;
        }
        const uint8_t *ra = sig + a * row_bytes, *rb = sig + b * row_bytes;
        uint32_t cnt = 0;
        if (VEC) {
            const uint4 *va = reinterpret_cast<const uint4 *>(ra), *vb = reinterpret_cast<const uint4 *>(rb);
            const int64_t nv = row_bytes / 16;
            for (int64_t i = lane; i < nv; i += 32) {
                uint4 x = __ldg(va + i), y = __ldg(vb + i);
                uint32_t d[4] = {x.x ^ y.x, x.y ^ y.y, x.z ^ y.z, x.w ^ y.w};
#pragma unroll
                for (int q = 0; q < 4; q++) {
                    if (SIGB == 2) cnt += ((d[q] & 0xFFFFu) == 0) + ((d[q] >> 16) == 0);
                    else cnt += ((d[q] & 0xFFu) == 0) + (((d[q] >> 8) & 0xFFu) == 0) + (((d[q] >> 16) & 0xFFu) == 0) +
                                ((d[q] >> 24) == 0);
                }
            }
        } else {
            for (uint32_t j = lane; j < k; j += 32) {
                if (SIGB == 2) cnt += reinterpret_cast<const uint16_t *>(ra)[j] == reinterpret_cast<const uint16_t *>(rb)[j];
                else cnt += ra[j] == rb[j];
            }
        }
        for (int o = 16; o; o >>= 1) cnt += __shfl_xor_sync(0xFFFFFFFFu, cnt, o);
        if (lane == 0) {
            matches[p] = cnt;
            if (jhat) jhat[p] = __fdiv_rn((float)cnt, (float)k);    // Eq. 14: J-hat = matches / k
        }
    }
}

}  // namespace wmh

using namespace wmh;

static wmh_status validate_hash(const wmh_layout *L, const wmh_rows *rows, uint32_t k, uint32_t cap,
                                int32_t sig_bytes, void *sig_out, bool host) {
    if (!L) { set_error("wmh_hash: layout is NULL"); return WMH_EINVAL; }
    wmh_status st = check_rows(rows, true);
    if (st != WMH_OK) return st;
    if (rows->dim != L->dim) { set_error("wmh_hash: rows dim %lld != layout dim %lld", (long long)rows->dim, (long long)L->dim); return WMH_EINVAL; }
    if (k < 1) { set_error("wmh_hash: k must be >= 1"); return WMH_EINVAL; }
    if (sig_bytes != 1 && sig_bytes != 2) { set_error("wmh_hash: sig_bytes=%d not in {1,2}", (int)sig_bytes); return WMH_EINVAL; }
    uint32_t maxcap = sig_bytes == 1 ? 255u : 65535u;
    if (cap < 1 || cap > maxcap) { set_error("wmh_hash: cap=%u outside [1, %u] for %d-byte signatures", cap, maxcap, (int)sig_bytes); return WMH_EINVAL; }
    if (rows->n_rows > 0 && !sig_out) { set_error("wmh_hash: sig_out is NULL"); return WMH_EINVAL; }
    if ((unsigned long long)rows->n_rows * k >= (1ull << 40)) { set_error("wmh_hash: n_rows*k too large"); return WMH_EINVAL; }
    (void)host;
    return WMH_OK;
}

static wmh_status hash_dispatch(const wmh_layout *L, const wmh_rows *rows, uint64_t seed, uint32_t k, uint32_t cap,
                                int32_t sig_bytes, void *sig_out, uint64_t *n_saturated, int algo, int chunk, cudaStream_t s,
                                int *algo_used) {
    *algo_used = algo == WMH_ALGO_AUTO ? WMH_ALGO_SIMPLE : algo;
    if (rows->n_rows == 0) return WMH_OK;
    HashArgs a;
    a.L = L;
    a.rows = *rows;
    a.S = splitmix64(seed);
    a.k = k;
    a.cap = cap;
    a.sig_bytes = sig_bytes;
    a.sig = sig_out;
    a.n_sat = reinterpret_cast<unsigned long long *>(n_saturated);
    a.stream = s;
    a.chunk = chunk;
    if (algo == WMH_ALGO_AUTO || algo == WMH_ALGO_TILED) {
        bool handled = false;
        wmh_status st = launch_hash_tiled(a, &handled);
        if (handled) *algo_used = WMH_ALGO_TILED;
        if (st != WMH_OK || handled) return st;
        if (algo == WMH_ALGO_TILED) { set_error("wmh_hash: the tiled kernel does not take this input shape"); return WMH_EINVAL; }
    }
    *algo_used = WMH_ALGO_SIMPLE;
    return launch_hash_simple(a);
}

extern "C" wmh_status wmh_hash_ex(const wmh_layout *L, const wmh_rows *rows, uint64_t seed, uint32_t k, uint32_t cap,
                                  int32_t sig_bytes, void *sig_out, uint64_t *n_saturated, wmh_hash_opts *opts,
                                  void *stream) {
    wmh_status st = validate_hash(L, rows, k, cap, sig_bytes, sig_out, false);
    if (st != WMH_OK) return st;
    int algo = WMH_ALGO_AUTO, chunk = 0;
    if (opts) {
        algo = opts->algo;
        for (int i = 0; i < 5; i++)
            if (opts->reserved[i]) { set_error("wmh_hash_ex: reserved option fields must be zero"); return WMH_EINVAL; }
        chunk = opts->chunk;
        if (chunk != 0 && chunk != 4 && chunk != 8 && chunk != 16 && chunk != 32) { set_error("wmh_hash_ex: chunk=%d not in {0,4,8,16,32}", chunk); return WMH_EINVAL; }
        if (algo < WMH_ALGO_AUTO || algo > WMH_ALGO_TILED) { set_error("wmh_hash_ex: unknown algo %d", algo); return WMH_EINVAL; }
    }
    int used = 0;
    st = hash_dispatch(L, rows, seed, k, cap, sig_bytes, sig_out, n_saturated, algo, chunk, (cudaStream_t)stream, &used);
    if (opts) opts->algo_used = used;
    return st;
}

extern "C" wmh_status wmh_hash(const wmh_layout *L, const wmh_rows *rows, uint64_t seed, uint32_t k, uint32_t cap,
                               int32_t sig_bytes, void *sig_out, uint64_t *n_saturated, void *stream) {
    return wmh_hash_ex(L, rows, seed, k, cap, sig_bytes, sig_out, n_saturated, nullptr, stream);
}

// ------------------------------------------------------------- e2e entry
namespace {
struct HostScratch {
    void *buf = nullptr;
    size_t bytes = 0;
    int device = -1;
    ~HostScratch() { if (buf) cudaFree(buf); }
    void *get(size_t need, wmh_status *st) {
        int dev = 0;
        cudaGetDevice(&dev);
        if (buf && (bytes < need || dev != device)) { cudaFree(buf); buf = nullptr; bytes = 0; }
        if (!buf) {
            size_t want = need + need / 8 + 256;
            if (cudaMalloc(&buf, want) != cudaSuccess) { *st = cuda_fail(cudaGetLastError(), "e2e scratch alloc"); return nullptr; }
            bytes = want;
            device = dev;
        }
        *st = WMH_OK;
        return buf;
    }
};
thread_local HostScratch g_scratch;
inline size_t align256(size_t v) { return (v + 255) & ~(size_t)255; }
}  // namespace

extern "C" wmh_status wmh_hash_host(const wmh_layout *L, const wmh_rows *rows_host, uint64_t seed, uint32_t k,
                                    uint32_t cap, int32_t sig_bytes, void *sig_out_host, void *stream) {
    wmh_status st = validate_hash(L, rows_host, k, cap, sig_bytes, sig_out_host, true);
    if (st != WMH_OK) return st;
    cudaStream_t s = (cudaStream_t)stream;
    const wmh_rows &h = *rows_host;
    if (h.n_rows == 0) return WMH_OK;
    size_t sig_bytes_total = (size_t)h.n_rows * k * sig_bytes;
    size_t in_bytes = 0, off_rp = 0, off_col = 0, off_val = 0;
    if (h.kind == WMH_DENSE) {
        in_bytes = align256((size_t)h.n_rows * h.dim);
    } else {
        off_rp = 0;
        off_col = align256(sizeof(int64_t) * (h.n_rows + 1));
        off_val = off_col + align256(sizeof(int32_t) * h.nnz);
        in_bytes = off_val + align256(h.nnz);
    }
    uint8_t *base = (uint8_t *)g_scratch.get(in_bytes + sig_bytes_total, &st);
    if (!base) return st;
    wmh_rows d = h;
    if (h.kind == WMH_DENSE) {
        WMH_CUDA_TRY(cudaMemcpyAsync(base, h.dense, (size_t)h.n_rows * h.dim, cudaMemcpyHostToDevice, s), "e2e H2D rows");
        d.dense = base;
    } else {
        WMH_CUDA_TRY(cudaMemcpyAsync(base + off_rp, h.row_ptr, sizeof(int64_t) * (h.n_rows + 1), cudaMemcpyHostToDevice, s), "e2e H2D row_ptr");
        if (h.nnz) {
            WMH_CUDA_TRY(cudaMemcpyAsync(base + off_col, h.col, sizeof(int32_t) * h.nnz, cudaMemcpyHostToDevice, s), "e2e H2D col");
            WMH_CUDA_TRY(cudaMemcpyAsync(base + off_val, h.val, h.nnz, cudaMemcpyHostToDevice, s), "e2e H2D val");
        }
        d.row_ptr = (const int64_t *)(base + off_rp);
        d.col = (const int32_t *)(base + off_col);
        d.val = base + off_val;
    }
    void *dsig = base + in_bytes;
    int used = 0;
    st = hash_dispatch(L, &d, seed, k, cap, sig_bytes, dsig, nullptr, WMH_ALGO_AUTO, 0, s, &used);
    if (st != WMH_OK) return st;
    WMH_CUDA_TRY(cudaMemcpyAsync(sig_out_host, dsig, sig_bytes_total, cudaMemcpyDeviceToHost, s), "e2e D2H signatures");
    WMH_CUDA_TRY(cudaStreamSynchronize(s), "e2e synchronize");
    return WMH_OK;
}

extern "C" wmh_status wmh_collide(const void *sig, int32_t sig_bytes, uint32_t k, int64_t n_rows, const int64_t *pairs,
                                  int64_t n_pairs, uint32_t *matches, float *jhat, int32_t check_pairs, void *stream) {
    if (sig_bytes != 1 && sig_bytes != 2) { set_error("wmh_collide: sig_bytes=%d not in {1,2}", (int)sig_bytes); return WMH_EINVAL; }
    if (k < 1) { set_error("wmh_collide: k must be >= 1"); return WMH_EINVAL; }
    if (n_pairs < 0 || n_rows < 0) { set_error("wmh_collide: negative sizes"); return WMH_EINVAL; }
    if (n_pairs == 0) return WMH_OK;
    if (!sig || !pairs || !matches) { set_error("wmh_collide: NULL pointer"); return WMH_EINVAL; }
    cudaStream_t s = (cudaStream_t)stream;
    unsigned long long *bad = nullptr;
    if (check_pairs) {
        WMH_CUDA_TRY(cudaMallocAsync((void **)&bad, sizeof(unsigned long long), s), "collide scratch");
        WMH_CUDA_TRY(cudaMemsetAsync(bad, 0, sizeof(unsigned long long), s), "collide scratch memset");
    }
    const bool vec = (((uintptr_t)sig) % 16 == 0) && (((int64_t)k * sig_bytes) % 16 == 0);
    const int threads = 256;
    int64_t blocks = min((int64_t)num_sms() * 16, (n_pairs * 32 + threads - 1) / threads);
    const uint8_t *sg = (const uint8_t *)sig;
#define WMH_COLLIDE(SB, V) collide_kernel<SB, V><<<(unsigned)blocks, threads, 0, s>>>(sg, k, n_rows, pairs, n_pairs, matches, jhat, bad)
    if (sig_bytes == 2) { if (vec) WMH_COLLIDE(2, true); else WMH_COLLIDE(2, false); }
    else { if (vec) WMH_COLLIDE(1, true); else WMH_COLLIDE(1, false); }
#undef WMH_COLLIDE
    WMH_LAUNCH_CHECK("collide launch");
    if (check_pairs) {
        unsigned long long nb = 0;
        cudaError_t e1 = cudaMemcpyAsync(&nb, bad, sizeof nb, cudaMemcpyDeviceToHost, s);
        cudaError_t e2 = cudaStreamSynchronize(s);
        cudaFreeAsync(bad, s);
        if (e1 != cudaSuccess || e2 != cudaSuccess) return cuda_fail(e1 != cudaSuccess ? e1 : e2, "collide readback");
        if (nb) { set_error("wmh_collide: %llu pairs index rows outside [0, %lld)", nb, (long long)n_rows); return WMH_EINVAL; }
    }
    return WMH_OK;
}

extern "C" const char *wmh_last_error(void) { return g_err; }

extern "C" const char *wmh_version(void) { return "wmh 0.1 sm_100a"; }
