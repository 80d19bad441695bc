// api.cu -- the C ABI (include/wmh.h): argument validation, hash dispatch, the
// host-buffer e2e entry, collide (a10, Eq. 14-15) and error reporting.
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <chrono>
#include <atomic>
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
    (void)cudaGetLastError();                    // a non-sticky error must not resurface in the next call's check
    return e == cudaErrorMemoryAllocation ? WMH_ENOMEM : WMH_ECUDA;
}

static std::atomic<unsigned long long> g_launches{0};

// ---- optional event bracket around the dominant kernel of a hash call
struct KernelTimer {
    bool on = false;
    int device = -1;
    cudaEvent_t a = nullptr, b = nullptr;
    bool recorded = false;
};
static thread_local KernelTimer g_ktimer;

void kernel_timer_begin(cudaStream_t s) {
    KernelTimer &t = g_ktimer;
    if (!t.on) return;
    int dev = 0;
    cudaGetDevice(&dev);
    if (t.device != dev) {
        if (t.a) { cudaEventDestroy(t.a); cudaEventDestroy(t.b); }
        cudaEventCreate(&t.a);
        cudaEventCreate(&t.b);
        t.device = dev;
    }
    cudaEventRecord(t.a, s);
}

void kernel_timer_end(cudaStream_t s) {
    KernelTimer &t = g_ktimer;
    if (!t.on || !t.b) return;
    cudaEventRecord(t.b, s);
    t.recorded = true;
}
void count_launch(unsigned n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

int num_sms() {
    static int cached[64] = {0};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
    if (!cached[dev]) {
        int v = 0;
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        cached[dev] = v > 0 ? v : 148;
        // The per-call scratch (draw tables, counters) comes from the device's
        // default stream-ordered pool; keep freed blocks in the pool instead of
        // returning them to the driver at every synchronisation, so a call never
        // pays a re-map (seen as occasional 1-2 ms step outliers).
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
            uint64_t keep = ~0ull;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
        }
    }
    return cached[dev];
}

wmh_status check_rows(const wmh_rows *rows, bool need_data) {
    if (!rows) { set_error("rows is NULL"); return WMH_EINVAL; }
    if (rows->n_rows < 0) { set_error("n_rows=%lld < 0", (long long)rows->n_rows); return WMH_EINVAL; }
    if (rows->dim < 1) { set_error("dim=%lld < 1", (long long)rows->dim); return WMH_EINVAL; }
    if (rows->weight_bytes < 0 || rows->weight_bytes > 2) { set_error("weight_bytes=%d not in {1, 2}", (int)rows->weight_bytes); return WMH_EINVAL; }
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
__global__ void __launch_bounds__(256) collide_kernel(const uint8_t *__restrict__ sig_a, int64_t n_a,
                                                      const uint8_t *__restrict__ sig_b, int64_t n_b, uint32_t k,
                                                      const int64_t *__restrict__ pairs, int64_t n_pairs,
                                                      uint32_t *__restrict__ matches, float *__restrict__ jhat,
                                                      unsigned long long *__restrict__ n_bad) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int64_t row_bytes = (int64_t)k * SIGB;
    for (int64_t p = warp; p < n_pairs; p += nwarps) {
        const int64_t a = __ldg(pairs + 2 * p), b = __ldg(pairs + 2 * p + 1);
        if (a < 0 || b < 0 || a >= n_a || b >= n_b) {
            if (lane == 0) {
                matches[p] = 0;
                if (jhat) jhat[p] = __int_as_float(0x7fc00000);
                if (n_bad) atomicAdd(n_bad, 1ull);
            }
            continue;
        }
        const uint8_t *ra = sig_a + a * row_bytes, *rb = sig_b + b * row_bytes;
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

static bool tiny_batch(const wmh_layout *L, const wmh_rows *rows, uint32_t k, uint32_t cap) {
    const double ed = L->mean_s > 0.0 ? std::min((double)cap, 1.0 / L->mean_s)
                                      : (rows->kind == WMH_CSR ? (double)cap : 32.0);
    return (unsigned long long)rows->n_rows * k <= (1ull << 20) &&
           (double)rows->n_rows * (double)k * ed <= (double)(1ull << 24);
}

static wmh_status hash_dispatch(const wmh_layout *L, const wmh_rows *rows, uint64_t seed, uint32_t k, uint32_t cap,
                                int32_t sig_bytes, void *sig_out, uint64_t *n_saturated, int algo, int chunk,
                                uint32_t horizon, cudaStream_t s, int *algo_used, int tile = 0, void *plan_out = nullptr,
                                int *tile_used = nullptr, bool bsearch = false) {
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
    a.horizon = horizon;
    a.tile = tile;
    a.plan_out = plan_out;
    a.tile_used = tile_used;
    a.isgreen_bsearch = bsearch;
    if (algo == WMH_ALGO_INDEX) {
        *algo_used = WMH_ALGO_INDEX;
        return launch_hash_index(a, horizon);
    }
    // tiny batches are launch-bound: the single-launch SIMPLE kernel beats the
    // table + tiled pair there (c1).  "Tiny" counts expected draws, not pairs
    // (Theorem 2: ~1/s per hash, s from prepare's statistics): a few sparse rows
    // at s ~ 1e-4 are 10^4 draws per hash, far cheaper on the index
    const bool tiny = tiny_batch(L, rows, k, cap);
    // The index kernel visits only the green draws (k*T*s per row); the tile
    // tests ~k/s draws per row, 4 rows per shared load.  Measured: CSR rows
    // (c3, c4) 35-350x faster on the index; dense rows at s = 0.05 (c2) 1.4x
    // and at s = 0.036 (c5) 1.2x faster on the tile.  Dense rows go to the index
    // only below mean s = 0.01 (prepare's statistics), where k/s tests dominate.
    const bool sparse_dense = rows->kind == WMH_DENSE && L->mean_s >= 0.0 && L->mean_s < 0.01;
    // uint16 weights / bounds above 255 (fixed-point real data): index or simple
    const bool wide = (L->flags & WMH_LAYOUT_WIDE) || weight_bytes(*rows) != 1;
    if (algo == WMH_ALGO_AUTO && !tiny && (rows->kind == WMH_CSR || sparse_dense || wide) &&
        index_feasible(L, k, cap, horizon)) {
        *algo_used = WMH_ALGO_INDEX;
        return launch_hash_index(a, horizon);
    }
    if (algo == WMH_ALGO_TILED || (algo == WMH_ALGO_AUTO && !tiny)) {
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
    int algo = WMH_ALGO_AUTO, chunk = 0, tile = 0;
    uint32_t horizon = 0;
    if (opts) {
        algo = opts->algo;
        const uint32_t tiles = WMH_OPT_TILE_BYTES | WMH_OPT_TILE_BITPLANES | WMH_OPT_TILE_BITSLICE;
        if (opts->flags & ~(uint32_t)(WMH_OPT_TIME_KERNEL | WMH_OPT_VALIDATE | WMH_OPT_ISGREEN_BINSEARCH | tiles)) { set_error("wmh_hash_ex: unknown flags 0x%x", opts->flags); return WMH_EINVAL; }
        if (__builtin_popcount(opts->flags & tiles) > 1) { set_error("wmh_hash_ex: the WMH_OPT_TILE_* flags are exclusive"); return WMH_EINVAL; }
        tile = (opts->flags & WMH_OPT_TILE_BYTES) ? 1 : (opts->flags & WMH_OPT_TILE_BITPLANES) ? 2
             : (opts->flags & WMH_OPT_TILE_BITSLICE) ? 3 : 0;
        for (int i = 0; i < 3; i++)
            if (opts->reserved[i]) { set_error("wmh_hash_ex: reserved option fields must be zero"); return WMH_EINVAL; }
        opts->tile_used = 0;
        chunk = opts->chunk;
        horizon = opts->horizon;
        if (chunk != 0 && chunk != 4 && chunk != 8 && chunk != 16 && chunk != 32) { set_error("wmh_hash_ex: chunk=%d not in {0,4,8,16,32}", chunk); return WMH_EINVAL; }
        if (algo < WMH_ALGO_AUTO || algo > WMH_ALGO_INDEX) { set_error("wmh_hash_ex: unknown algo %d", algo); return WMH_EINVAL; }
    }
    if (opts && (opts->flags & WMH_OPT_VALIDATE)) {
        st = wmh_check_rows(L, rows, stream);
        if (st != WMH_OK) return st;
    }
    int used = 0;
    g_ktimer.on = opts && (opts->flags & WMH_OPT_TIME_KERNEL);
    if (g_ktimer.on) g_ktimer.recorded = false;
    st = hash_dispatch(L, rows, seed, k, cap, sig_bytes, sig_out, n_saturated, algo, chunk, horizon, (cudaStream_t)stream,
                       &used, tile, opts ? opts->plan_out : nullptr, opts ? &opts->tile_used : nullptr,
                       opts && (opts->flags & WMH_OPT_ISGREEN_BINSEARCH));
    g_ktimer.on = false;
    if (opts) {
        opts->algo_used = used;
        if (used == WMH_ALGO_INDEX) opts->horizon = index_horizon(L, k, cap, horizon);   // the T it filed
    }
    return st;
}

// ---- a prepared hash family: the index built once, many row batches
struct wmh_hasher {
    const wmh_layout *L = nullptr;
    uint64_t seed = 0;
    uint32_t k = 0, cap = 0;
    IndexBuilt ix;
    cudaEvent_t built = nullptr;     // recorded after the build on the create stream
};

extern "C" wmh_status wmh_hasher_create(const wmh_layout *L, uint64_t seed, uint32_t k, uint32_t cap, uint32_t horizon,
                                        wmh_hasher **out, void *stream) {
    if (!out) { set_error("wmh_hasher_create: out is NULL"); return WMH_EINVAL; }
    *out = nullptr;
    if (!L) { set_error("wmh_hasher_create: layout is NULL"); return WMH_EINVAL; }
    if (k < 1 || k > 65536) { set_error("wmh_hasher_create: k=%u not in [1, 65536]", k); return WMH_EINVAL; }
    if (cap < 1 || cap > 65535) { set_error("wmh_hasher_create: cap=%u not in [1, 65535]", cap); return WMH_EINVAL; }
    HashArgs a{};
    a.L = L;
    a.S = splitmix64(seed);
    a.k = k;
    a.cap = cap;
    a.stream = (cudaStream_t)stream;
    wmh_hasher *h = new wmh_hasher();
    h->L = L;
    h->seed = seed;
    h->k = k;
    h->cap = cap;
    wmh_status st = index_build(a, horizon, &h->ix);
    if (st != WMH_OK) { delete h; return st; }
    if (cudaEventCreateWithFlags(&h->built, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventRecord(h->built, a.stream) != cudaSuccess) {
        const cudaError_t e = cudaGetLastError();
        index_free(h->ix, a.stream);
        if (h->built) cudaEventDestroy(h->built);
        delete h;
        return cuda_fail(e, "wmh_hasher_create event");
    }
    *out = h;
    return WMH_OK;
}

extern "C" wmh_status wmh_hasher_run(const wmh_hasher *h, const wmh_rows *rows, int32_t sig_bytes, void *sig_out,
                                     uint64_t *n_saturated, void *stream) {
    if (!h) { set_error("wmh_hasher_run: hasher is NULL"); return WMH_EINVAL; }
    wmh_status st = validate_hash(h->L, rows, h->k, h->cap, sig_bytes, sig_out, false);
    if (st != WMH_OK) return st;
    if (rows->n_rows == 0) return WMH_OK;
    HashArgs a{};
    a.L = h->L;
    a.rows = *rows;
    a.S = splitmix64(h->seed);
    a.k = h->k;
    a.cap = h->cap;
    a.sig_bytes = sig_bytes;
    a.sig = sig_out;
    a.n_sat = reinterpret_cast<unsigned long long *>(n_saturated);
    a.stream = (cudaStream_t)stream;
    // runs on any stream see the finished build (create may have used another)
    WMH_CUDA_TRY(cudaStreamWaitEvent(a.stream, h->built, 0), "wmh_hasher_run wait for the build");
    return index_rows(a, h->ix);
}

extern "C" void wmh_hasher_free(wmh_hasher *h) {
    if (!h) return;
    if (h->ix.scr) cudaFree(h->ix.scr);          // (pool memory: cudaFree synchronises)
    if (h->built) cudaEventDestroy(h->built);
    delete h;
}

extern "C" wmh_status wmh_hash(const wmh_layout *L, const wmh_rows *rows, uint64_t seed, uint32_t k, uint32_t cap,
                               int32_t sig_bytes, void *sig_out, uint64_t *n_saturated, void *stream) {
    return wmh_hash_ex(L, rows, seed, k, cap, sig_bytes, sig_out, n_saturated, nullptr, stream);
}

// ------------------------------------------------------------- e2e entry
// Host rows in, host signatures out.  The rows are cut into chunks that flow
// through three internal streams -- H2D copy, hash, D2H copy -- so the PCIe
// transfers of neighbouring chunks overlap each other and the kernels.
namespace {
constexpr int E2E_SLOTS = 3;
constexpr int E2E_CHUNKS = 8;

struct E2EState {
    int device = -1;
    cudaStream_t s_in = nullptr, s_comp = nullptr, s_out = nullptr;
    cudaEvent_t ev_start = nullptr, ev_in[E2E_SLOTS] = {}, ev_comp[E2E_SLOTS] = {}, ev_out[E2E_SLOTS] = {};
    void *buf[E2E_SLOTS] = {};
    size_t bytes[E2E_SLOTS] = {};

    wmh_status init() {
        int dev = 0;
        cudaGetDevice(&dev);
        if (device == dev) return WMH_OK;
        release();
        WMH_CUDA_TRY(cudaStreamCreateWithFlags(&s_in, cudaStreamNonBlocking), "e2e stream");
        WMH_CUDA_TRY(cudaStreamCreateWithFlags(&s_comp, cudaStreamNonBlocking), "e2e stream");
        WMH_CUDA_TRY(cudaStreamCreateWithFlags(&s_out, cudaStreamNonBlocking), "e2e stream");
        WMH_CUDA_TRY(cudaEventCreateWithFlags(&ev_start, cudaEventDisableTiming), "e2e event");
        for (int i = 0; i < E2E_SLOTS; i++) {
            WMH_CUDA_TRY(cudaEventCreateWithFlags(&ev_in[i], cudaEventDisableTiming), "e2e event");
            WMH_CUDA_TRY(cudaEventCreateWithFlags(&ev_comp[i], cudaEventDisableTiming), "e2e event");
            WMH_CUDA_TRY(cudaEventCreateWithFlags(&ev_out[i], cudaEventDisableTiming), "e2e event");
        }
        device = dev;
        return WMH_OK;
    }
    wmh_status reserve(int slot, size_t need) {
        if (bytes[slot] >= need) return WMH_OK;
        if (buf[slot]) { cudaStreamSynchronize(s_out); cudaFree(buf[slot]); buf[slot] = nullptr; bytes[slot] = 0; }
        WMH_CUDA_TRY(cudaMalloc(&buf[slot], need), "e2e scratch alloc");
        bytes[slot] = need;
        return WMH_OK;
    }
    void release() {
        if (device < 0) return;
        for (int i = 0; i < E2E_SLOTS; i++) {
            if (buf[i]) cudaFree(buf[i]);
            buf[i] = nullptr;
            bytes[i] = 0;
            if (ev_in[i]) cudaEventDestroy(ev_in[i]);
            if (ev_comp[i]) cudaEventDestroy(ev_comp[i]);
            if (ev_out[i]) cudaEventDestroy(ev_out[i]);
        }
        if (ev_start) cudaEventDestroy(ev_start);
        if (s_in) cudaStreamDestroy(s_in);
        if (s_comp) cudaStreamDestroy(s_comp);
        if (s_out) cudaStreamDestroy(s_out);
        device = -1;
    }
    ~E2EState() { release(); }
};
thread_local E2EState g_e2e;
inline size_t align256(size_t v) { return (v + 255) & ~(size_t)255; }

__global__ void rebase_row_ptr(int64_t *rp, int64_t n, int64_t base) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        rp[i] -= base;
}
}  // namespace

extern "C" wmh_status wmh_hash_host(const wmh_layout *L, const wmh_rows *rows_host, uint64_t seed, uint32_t k,
                                    uint32_t cap, int32_t sig_bytes, void *sig_out_host, void *stream) {
    wmh_status st = validate_hash(L, rows_host, k, cap, sig_bytes, sig_out_host, true);
    if (st != WMH_OK) return st;
    const wmh_rows &h = *rows_host;
    if (h.n_rows == 0) return WMH_OK;
    E2EState &E = g_e2e;
    if ((st = E.init()) != WMH_OK) return st;
    // Chunk boundaries.  The copies of the first chunk in and the last chunk out
    // are not overlapped by anything, so large batches ramp: chunk sizes in the
    // proportions 1 2 4 4 4 4 4 4 2 1 (measured on c2: 2.85 ms with 8 equal
    // chunks against a 2.2 ms PCIe bound); smaller batches use <= E2E_CHUNKS
    // equal chunks of >= 2048 rows.  WMH_E2E_CHUNKS=n forces n equal chunks.
    static const int env_chunks = getenv("WMH_E2E_CHUNKS") ? atoi(getenv("WMH_E2E_CHUNKS")) : 0;
    std::vector<int64_t> cut{0};
    {
        static const int ramp[] = {1, 2, 4, 4, 4, 4, 4, 4, 2, 1};
        constexpr int n_ramp = (int)(sizeof ramp / sizeof ramp[0]);
        int wsum = 0;
        for (int i = 0; i < n_ramp; i++) wsum += ramp[i];
        if (env_chunks <= 0 && h.n_rows >= (int64_t)wsum * 2048) {
            int acc = 0;
            for (int i = 0; i < n_ramp; i++) {
                acc += ramp[i];
                cut.push_back(h.n_rows * acc / wsum);
            }
        } else {
            const int64_t max_chunks = env_chunks > 0 ? env_chunks : E2E_CHUNKS;
            const int64_t cr = std::max<int64_t>(2048, (h.n_rows + max_chunks - 1) / max_chunks);
            for (int64_t b = cr; b < h.n_rows + cr; b += cr) cut.push_back(std::min<int64_t>(b, h.n_rows));
        }
    }
    const int64_t n_chunks = (int64_t)cut.size() - 1;
    // WMH_E2E_TRACE=1: per-chunk stage times on stderr (timing events; diagnostics only)
    static const bool trace = getenv("WMH_E2E_TRACE") != nullptr;
    std::vector<cudaEvent_t> tev;
    auto tmark = [&](cudaStream_t st_) {
        if (!trace) return;
        cudaEvent_t e;
        cudaEventCreate(&e);
        cudaEventRecord(e, st_);
        tev.push_back(e);
    };
    const auto host_t0 = std::chrono::steady_clock::now();
    tmark((cudaStream_t)stream);
    const size_t row_sig = (size_t)k * sig_bytes;
    WMH_CUDA_TRY(cudaEventRecord(E.ev_start, (cudaStream_t)stream), "e2e start event");
    WMH_CUDA_TRY(cudaStreamWaitEvent(E.s_in, E.ev_start, 0), "e2e wait");
    WMH_CUDA_TRY(cudaStreamWaitEvent(E.s_comp, E.ev_start, 0), "e2e wait");
    // the index kernel (AUTO's choice for CSR rows) files the draws once for the
    // whole call; every chunk then only runs its rows kernel
    const bool use_index = (h.kind == WMH_CSR || (L->mean_s >= 0.0 && L->mean_s < 0.01) ||
                            (L->flags & WMH_LAYOUT_WIDE) || weight_bytes(h) != 1) && index_feasible(L, k, cap, 0) &&
                           !tiny_batch(L, &h, k, cap);
    IndexBuilt ix;
    struct IxGuard {                             // frees the index on every return path
        IndexBuilt *ix;
        cudaStream_t s;
        ~IxGuard() { index_free(*ix, s); }
    } guard{&ix, E.s_comp};
    HashArgs ha;
    if (use_index) {
        ha.L = L;
        ha.rows = h;
        ha.S = splitmix64(seed);
        ha.k = k;
        ha.cap = cap;
        ha.sig_bytes = sig_bytes;
        ha.sig = nullptr;
        ha.n_sat = nullptr;
        ha.stream = E.s_comp;
        ha.chunk = 0;
        ha.horizon = 0;
        if ((st = index_build(ha, 0, &ix)) != WMH_OK) return st;
    }
    for (int64_t ci = 0; ci < n_chunks; ci++) {
        const int slot = (int)(ci % E2E_SLOTS);
        const int64_t a = cut[ci], b = cut[ci + 1], nr = b - a;
        size_t in_bytes, off_col = 0, off_val = 0;
        int64_t e0 = 0, e1 = 0;
        const size_t wb = (size_t)weight_bytes(h);
        if (h.kind == WMH_DENSE) {
            in_bytes = align256((size_t)nr * h.dim * wb);
        } else {
            e0 = h.row_ptr[a];
            e1 = h.row_ptr[b];
            off_col = align256(sizeof(int64_t) * (nr + 1));
            off_val = off_col + align256(sizeof(int32_t) * (e1 - e0));
            in_bytes = off_val + align256((size_t)(e1 - e0) * wb);
        }
        // the slot's previous chunk must have finished its D2H before reuse
        WMH_CUDA_TRY(cudaStreamWaitEvent(E.s_in, E.ev_out[slot], 0), "e2e wait");
        if ((st = E.reserve(slot, in_bytes + nr * row_sig)) != WMH_OK) return st;
        uint8_t *base = (uint8_t *)E.buf[slot];
        wmh_rows d = h;
        d.n_rows = nr;
        if (h.kind == WMH_DENSE) {
            WMH_CUDA_TRY(cudaMemcpyAsync(base, h.dense + a * h.dim * wb, (size_t)nr * h.dim * wb, cudaMemcpyHostToDevice, E.s_in), "e2e H2D rows");
            d.dense = base;
        } else {
            WMH_CUDA_TRY(cudaMemcpyAsync(base, h.row_ptr + a, sizeof(int64_t) * (nr + 1), cudaMemcpyHostToDevice, E.s_in), "e2e H2D row_ptr");
            if (e1 > e0) {
                WMH_CUDA_TRY(cudaMemcpyAsync(base + off_col, h.col + e0, sizeof(int32_t) * (e1 - e0), cudaMemcpyHostToDevice, E.s_in), "e2e H2D col");
                WMH_CUDA_TRY(cudaMemcpyAsync(base + off_val, h.val + e0 * wb, (size_t)(e1 - e0) * wb, cudaMemcpyHostToDevice, E.s_in), "e2e H2D val");
            }
            rebase_row_ptr<<<std::max<int64_t>(1, std::min<int64_t>(64, (nr + 256) / 256)), 256, 0, E.s_in>>>((int64_t *)base, nr + 1, e0);
            WMH_LAUNCH_CHECK("e2e rebase");
            d.row_ptr = (const int64_t *)base;
            d.col = (const int32_t *)(base + off_col);
            d.val = base + off_val;
            d.nnz = e1 - e0;
        }
        tmark(E.s_in);
        WMH_CUDA_TRY(cudaEventRecord(E.ev_in[slot], E.s_in), "e2e event");
        WMH_CUDA_TRY(cudaStreamWaitEvent(E.s_comp, E.ev_in[slot], 0), "e2e wait");
        void *dsig = base + in_bytes;
        if (use_index) {
            HashArgs ca = ha;
            ca.rows = d;
            ca.sig = dsig;
            st = index_rows(ca, ix);
        } else {
            int used = 0;
            st = hash_dispatch(L, &d, seed, k, cap, sig_bytes, dsig, nullptr, WMH_ALGO_AUTO, 0, 0, E.s_comp, &used);
        }
        if (st != WMH_OK) return st;
        tmark(E.s_comp);
        WMH_CUDA_TRY(cudaEventRecord(E.ev_comp[slot], E.s_comp), "e2e event");
        WMH_CUDA_TRY(cudaStreamWaitEvent(E.s_out, E.ev_comp[slot], 0), "e2e wait");
        WMH_CUDA_TRY(cudaMemcpyAsync((uint8_t *)sig_out_host + a * row_sig, dsig, nr * row_sig, cudaMemcpyDeviceToHost, E.s_out), "e2e D2H signatures");
        tmark(E.s_out);
        WMH_CUDA_TRY(cudaEventRecord(E.ev_out[slot], E.s_out), "e2e event");
    }
    const double host_us = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - host_t0).count();
    index_free(ix, E.s_comp);                    // stream-ordered after the last chunk's kernel
    WMH_CUDA_TRY(cudaStreamSynchronize(E.s_out), "e2e synchronize");
    if (trace && !tev.empty()) {
        cudaDeviceSynchronize();
        fprintf(stderr, "[wmh e2e] %lld chunks, host enqueue %.0f us; per chunk (in, comp, out) end ms:", (long long)n_chunks,
                host_us);
        for (size_t i = 1; i < tev.size(); i++) {
            float ms = 0.f;
            cudaEventElapsedTime(&ms, tev[0], tev[i]);
            fprintf(stderr, "%s%.3f", (i - 1) % 3 == 0 ? " | " : " ", ms);
        }
        fprintf(stderr, "\n");
        for (cudaEvent_t e : tev) cudaEventDestroy(e);
    }
    return WMH_OK;
}

static wmh_status collide_impl(const char *who, const void *sig_a, int64_t n_a, const void *sig_b, int64_t n_b,
                               int32_t sig_bytes, uint32_t k, const int64_t *pairs, int64_t n_pairs, uint32_t *matches,
                               float *jhat, int32_t check_pairs, void *stream) {
    if (sig_bytes != 1 && sig_bytes != 2) { set_error("%s: sig_bytes=%d not in {1,2}", who, (int)sig_bytes); return WMH_EINVAL; }
    if (k < 1) { set_error("%s: k must be >= 1", who); return WMH_EINVAL; }
    if (n_pairs < 0 || n_a < 0 || n_b < 0) { set_error("%s: negative sizes", who); return WMH_EINVAL; }
    if (n_pairs == 0) return WMH_OK;
    if (!sig_a || !sig_b || !pairs || !matches) { set_error("%s: NULL pointer", who); return WMH_EINVAL; }
    cudaStream_t s = (cudaStream_t)stream;
    unsigned long long *bad = nullptr;
    if (check_pairs) {
        WMH_CUDA_TRY(cudaMallocAsync((void **)&bad, sizeof(unsigned long long), s), "collide scratch");
        WMH_CUDA_TRY(cudaMemsetAsync(bad, 0, sizeof(unsigned long long), s), "collide scratch memset");
    }
    const bool vec = (((uintptr_t)sig_a) % 16 == 0) && (((uintptr_t)sig_b) % 16 == 0) && (((int64_t)k * sig_bytes) % 16 == 0);
    const int threads = 256;
    int64_t blocks = min((int64_t)num_sms() * 16, (n_pairs * 32 + threads - 1) / threads);
    const uint8_t *ga = (const uint8_t *)sig_a, *gb = (const uint8_t *)sig_b;
#define WMH_COLLIDE(SB, V) collide_kernel<SB, V><<<(unsigned)blocks, threads, 0, s>>>(ga, n_a, gb, n_b, k, pairs, n_pairs, matches, jhat, bad)
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
        if (nb) { set_error("%s: %llu pairs index rows outside [0, %lld) x [0, %lld)", who, nb, (long long)n_a, (long long)n_b); return WMH_EINVAL; }
    }
    return WMH_OK;
}

extern "C" wmh_status wmh_collide(const void *sig, int32_t sig_bytes, uint32_t k, int64_t n_rows, const int64_t *pairs,
                                  int64_t n_pairs, uint32_t *matches, float *jhat, int32_t check_pairs, void *stream) {
    return collide_impl("wmh_collide", sig, n_rows, sig, n_rows, sig_bytes, k, pairs, n_pairs, matches, jhat, check_pairs,
                        stream);
}

extern "C" wmh_status wmh_collide2(const void *sig_a, int64_t n_a, const void *sig_b, int64_t n_b, int32_t sig_bytes,
                                   uint32_t k, const int64_t *pairs, int64_t n_pairs, uint32_t *matches, float *jhat,
                                   int32_t check_pairs, void *stream) {
    return collide_impl("wmh_collide2", sig_a, n_a, sig_b, n_b, sig_bytes, k, pairs, n_pairs, matches, jhat, check_pairs,
                        stream);
}

namespace wmh {
__global__ void empty_kernel() {}
}  // namespace wmh

// The launch floor: one empty kernel on `stream` (what a launch- or graph-node-
// bound configuration such as c1 is measured against).
extern "C" wmh_status wmh_empty_launch(void *stream) {
    wmh::empty_kernel<<<1, 32, 0, (cudaStream_t)stream>>>();
    WMH_LAUNCH_CHECK("empty launch");
    return WMH_OK;
}

extern "C" const char *wmh_last_error(void) { return g_err; }

extern "C" const char *wmh_version(void) { return "wmh 0.1 sm_100a"; }

extern "C" uint64_t wmh_kernel_launches(void) { return wmh::g_launches.load(std::memory_order_relaxed); }

extern "C" wmh_status wmh_last_kernel_ms(float *ms) {
    if (!ms) { set_error("wmh_last_kernel_ms: ms is NULL"); return WMH_EINVAL; }
    KernelTimer &t = g_ktimer;
    if (!t.recorded) { set_error("wmh_last_kernel_ms: no timed hash call on this thread"); return WMH_EINVAL; }
    WMH_CUDA_TRY(cudaEventSynchronize(t.b), "kernel timer sync");
    WMH_CUDA_TRY(cudaEventElapsedTime(ms, t.a, t.b), "kernel timer elapsed");
    return WMH_OK;
}
