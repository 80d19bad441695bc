// lsh.cu -- f3: the (K, L) banding LSH index over the signatures (the
// paper's first listed consequence: weighted minwise hashing in constant time
// makes the (K, L)-parameterised LSH query O(KL + dL)).
//
// Band b of a signature row is its hashes [bK, (b+1)K).  Two rows collide in
// band b iff those K values are equal; the candidates of a query are the rows
// that collide with it in at least one band.  A pair with per-hash collision
// probability p (= J, Theorem 1) is a candidate with probability
// 1 - (1 - p^K)^L.
//
// Build (per band, on the device): a 32-bit key of the band's K values, an
// open-addressed table key -> bucket (atomicCAS, linear probing), bucket
// sizes, their exclusive scan, and the rows scattered into their buckets.
// Query (one warp per query row): for each band the bucket of the query's
// key; every row in it is checked against the query's band values (so key
// collisions never produce a false candidate) and against the earlier bands
// (a row is reported once, for its first colliding band).
#include <stdio.h>

#include <algorithm>

#include "common.cuh"

struct wmh_lsh {
    const void *sig = nullptr;   // caller-owned signatures (n_rows x k), kept alive by the caller
    int sig_bytes = 2;
    uint32_t k = 0, K = 0, L = 0;
    int64_t n_rows = 0;
    uint32_t cap_log2 = 0;       // table capacity per band = 2^cap_log2
    uint32_t *keys = nullptr;    // [L][cap]  bucket keys (EMPTY = 0xFFFFFFFF)
    uint32_t *start = nullptr;   // [L * cap + 1] bucket start (index into rows)
    int64_t *rows = nullptr;     // [L * n_rows] row ids, grouped by bucket
    uint8_t *scratch = nullptr;
    int device = 0;
};

namespace wmh {

constexpr uint32_t LSH_EMPTY = 0xFFFFFFFFu;

template <typename S>
__device__ __forceinline__ uint32_t lsh_key(const S *row, uint32_t b, uint32_t K) {
    uint64_t acc = 0x243F6A8885A308D3ull ^ b;            // band index as the salt
    for (uint32_t i = 0; i < K; i++) acc = splitmix64(acc ^ (uint64_t)row[b * K + i]);
    const uint32_t key = (uint32_t)(acc >> 32);
    return key == LSH_EMPTY ? LSH_EMPTY - 1 : key;
}

__device__ __forceinline__ uint32_t lsh_home(uint32_t key, uint32_t cap_log2) {
    return (key * 0x9E3779B1u) >> (32 - cap_log2);
}

// one thread per (band, row): key, bucket (insert), bucket size
template <typename S>
__global__ void lsh_insert_kernel(const S *__restrict__ sig, uint32_t k, int64_t n_rows, uint32_t K, uint32_t L,
                                  uint32_t cap_log2, uint32_t *__restrict__ keys, uint32_t *__restrict__ slot_of,
                                  uint32_t *__restrict__ count) {
    const uint32_t cap = 1u << cap_log2;
    const int64_t total = n_rows * (int64_t)L;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t b = (uint32_t)(i / n_rows);
        const int64_t n = i - (int64_t)b * n_rows;
        const uint32_t key = lsh_key(sig + n * k, b, K);
        uint32_t *tb = keys + (uint64_t)b * cap;
        uint32_t s = lsh_home(key, cap_log2);
        for (;;) {
            const uint32_t old = atomicCAS(tb + s, LSH_EMPTY, key);
            if (old == LSH_EMPTY || old == key) break;
            s = (s + 1) & (cap - 1);
        }
        slot_of[i] = s;
        atomicAdd(count + 1 + (uint64_t)b * cap + s, 1u);
    }
}

__global__ void lsh_scatter_kernel(int64_t n_rows, uint32_t L, uint32_t cap_log2, const uint32_t *__restrict__ slot_of,
                                   uint32_t *__restrict__ cursor, int64_t *__restrict__ rows) {
    const uint32_t cap = 1u << cap_log2;
    const int64_t total = n_rows * (int64_t)L;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t b = (uint32_t)(i / n_rows);
        const int64_t n = i - (int64_t)b * n_rows;
        rows[atomicAdd(cursor + (uint64_t)b * cap + slot_of[i], 1u)] = n;
    }
}

// one warp per query
template <typename S>
__global__ void lsh_query_kernel(const S *__restrict__ sig, uint32_t k, uint32_t K, uint32_t L, uint32_t cap_log2,
                                 const uint32_t *__restrict__ keys, const uint32_t *__restrict__ start,
                                 const int64_t *__restrict__ rows, const S *__restrict__ qsig, int64_t n_q,
                                 uint32_t max_out, int64_t *__restrict__ out_rows, uint32_t *__restrict__ out_count) {
    const int lane = threadIdx.x & 31;
    const uint32_t cap = 1u << cap_log2;
    const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t q = w0; q < n_q; q += nw) {
        const S *qr = qsig + q * k;
        uint32_t found = 0;
        for (uint32_t b = 0; b < L; b++) {
            const uint32_t key = lsh_key(qr, b, K);
            const uint32_t *tb = keys + (uint64_t)b * cap;
            uint32_t s = lsh_home(key, cap_log2), hit = LSH_EMPTY;
            for (;;) {                                       // probe (warp-uniform)
                const uint32_t kk = __ldg(tb + s);
                if (kk == key) { hit = s; break; }
                if (kk == LSH_EMPTY) break;
                s = (s + 1) & (cap - 1);
            }
            if (hit == LSH_EMPTY) continue;
            const uint32_t a = __ldg(start + (uint64_t)b * cap + hit), e = __ldg(start + (uint64_t)b * cap + hit + 1);
            for (uint32_t i0 = a; i0 < e; i0 += 32) {
                bool take = false;
                int64_t n = -1;
                if (i0 + lane < e) {
                    n = __ldg(rows + i0 + lane);
                    const S *rr = sig + n * k;
                    take = true;
                    for (uint32_t i = b * K; i < (b + 1) * K && take; i++) take = rr[i] == qr[i];   // band b equal
                    for (uint32_t b2 = 0; b2 < b && take; b2++) {                              // not seen earlier
                        bool same = true;
                        for (uint32_t i = b2 * K; i < (b2 + 1) * K && same; i++) same = rr[i] == qr[i];
                        take = !same;
                    }
                }
                const unsigned m = __ballot_sync(0xFFFFFFFFu, take);
                const uint32_t pos = found + __popc(m & ((1u << lane) - 1));
                if (take && pos < max_out && out_rows) out_rows[q * (int64_t)max_out + pos] = n;
                found += __popc(m);
            }
        }
        if (lane == 0) out_count[q] = found;
    }
}

}  // namespace wmh

using namespace wmh;

extern "C" void wmh_lsh_free(wmh_lsh *ix) {
    if (!ix) return;
    cudaFree(ix->scratch);
    delete ix;
}

extern "C" wmh_status wmh_lsh_build(const void *sig, int32_t sig_bytes, uint32_t k, int64_t n_rows, uint32_t K,
                                    uint32_t L, wmh_lsh **out, void *stream) {
    if (!out) { set_error("wmh_lsh_build: out is NULL"); return WMH_EINVAL; }
    *out = nullptr;
    if (sig_bytes != 1 && sig_bytes != 2) { set_error("wmh_lsh_build: sig_bytes=%d not in {1,2}", (int)sig_bytes); return WMH_EINVAL; }
    if (K < 1 || L < 1 || (uint64_t)K * L > k) { set_error("wmh_lsh_build: need K, L >= 1 and K*L <= k (K=%u L=%u k=%u)", K, L, k); return WMH_EINVAL; }
    if (n_rows < 1 || n_rows >= (1ll << 31) || (uint64_t)n_rows * L >= (1ull << 32)) { set_error("wmh_lsh_build: n_rows=%lld out of range", (long long)n_rows); return WMH_EINVAL; }
    if (!sig) { set_error("wmh_lsh_build: sig is NULL"); return WMH_EINVAL; }
    cudaStream_t s = (cudaStream_t)stream;
    wmh_lsh *ix = new wmh_lsh();
    ix->sig = sig;
    ix->sig_bytes = sig_bytes;
    ix->k = k;
    ix->K = K;
    ix->L = L;
    ix->n_rows = n_rows;
    uint32_t cl = 6;
    while ((1ull << cl) < 2ull * (uint64_t)n_rows) cl++;
    ix->cap_log2 = cl;
    const uint64_t cap = 1ull << cl;
    cudaGetDevice(&ix->device);
    auto al = [](uint64_t v) { return (v + 255) & ~(uint64_t)255; };
    const uint64_t keys_b = al(L * cap * 4), start_b = al((L * cap + 1) * 4), rows_b = al((uint64_t)L * n_rows * 8);
    const uint64_t slot_b = al((uint64_t)L * n_rows * 4);
    const int64_t nsc = (int64_t)((L * cap + 8191) / 8192);
    const uint64_t sums_b = al((uint64_t)nsc * 4 + 4);
    if (cudaMalloc((void **)&ix->scratch, keys_b + start_b + rows_b + slot_b + sums_b) != cudaSuccess) {
        delete ix;
        set_error("wmh_lsh_build: allocation of %llu bytes failed", (unsigned long long)(keys_b + start_b + rows_b + slot_b + sums_b));
        return WMH_ENOMEM;
    }
    ix->keys = reinterpret_cast<uint32_t *>(ix->scratch);
    ix->start = reinterpret_cast<uint32_t *>(ix->scratch + keys_b);
    ix->rows = reinterpret_cast<int64_t *>(ix->scratch + keys_b + start_b);
    uint32_t *slot_of = reinterpret_cast<uint32_t *>(ix->scratch + keys_b + start_b + rows_b);
    uint32_t *sums = reinterpret_cast<uint32_t *>(ix->scratch + keys_b + start_b + rows_b + slot_b);
    auto fail = [&](wmh_status st) { wmh_lsh_free(ix); return st; };
    if (cudaMemsetAsync(ix->keys, 0xFF, L * cap * 4, s) != cudaSuccess ||
        cudaMemsetAsync(ix->start, 0, (L * cap + 1) * 4, s) != cudaSuccess)
        return fail(cuda_fail(cudaGetLastError(), "lsh memset"));
    const int64_t total = n_rows * (int64_t)L;
    const int blocks = (int)std::min<int64_t>((int64_t)num_sms() * 16, (total + 255) / 256);
    if (sig_bytes == 2)
        lsh_insert_kernel<<<blocks, 256, 0, s>>>(reinterpret_cast<const uint16_t *>(sig), k, n_rows, K, L, cl, ix->keys,
                                                 slot_of, ix->start);
    else
        lsh_insert_kernel<<<blocks, 256, 0, s>>>(reinterpret_cast<const uint8_t *>(sig), k, n_rows, K, L, cl, ix->keys,
                                                 slot_of, ix->start);
    count_launch();
    if (cudaGetLastError() != cudaSuccess) return fail(cuda_fail(cudaGetLastError(), "lsh insert"));
    // start[b*cap + s] = rows in buckets before (b, s): inclusive scan of the sizes stored at +1
    wmh_status st = scan_u32_inplace(ix->start + 1, (int64_t)(L * cap), sums, s);
    if (st != WMH_OK) return fail(st);
    // the scatter advances start[b*cap + s] from the bucket's start to its end, so the
    // ranges are read from a copy taken before it: keep start, scatter through a cursor
    uint32_t *cursor = nullptr;
    if (cudaMallocAsync((void **)&cursor, (L * cap + 1) * 4, s) != cudaSuccess) return fail(WMH_ENOMEM);
    cudaMemcpyAsync(cursor, ix->start, (L * cap + 1) * 4, cudaMemcpyDeviceToDevice, s);
    lsh_scatter_kernel<<<blocks, 256, 0, s>>>(n_rows, L, cl, slot_of, cursor, ix->rows);
    count_launch();
    cudaFreeAsync(cursor, s);
    if (cudaGetLastError() != cudaSuccess) return fail(cuda_fail(cudaGetLastError(), "lsh scatter"));
    *out = ix;
    return WMH_OK;
}

extern "C" wmh_status wmh_lsh_query(const wmh_lsh *ix, const void *qsig, int64_t n_q, uint32_t max_out,
                                    int64_t *out_rows, uint32_t *out_count, void *stream) {
    if (!ix) { set_error("wmh_lsh_query: index is NULL"); return WMH_EINVAL; }
    if (n_q < 0) { set_error("wmh_lsh_query: n_q < 0"); return WMH_EINVAL; }
    if (n_q == 0) return WMH_OK;
    if (!qsig || !out_count || (max_out > 0 && !out_rows)) { set_error("wmh_lsh_query: NULL pointer"); return WMH_EINVAL; }
    cudaStream_t s = (cudaStream_t)stream;
    const int blocks = (int)std::min<int64_t>((int64_t)num_sms() * 16, (n_q * 32 + 255) / 256);
    if (ix->sig_bytes == 2)
        lsh_query_kernel<<<blocks, 256, 0, s>>>(reinterpret_cast<const uint16_t *>(ix->sig), ix->k, ix->K, ix->L,
                                                ix->cap_log2, ix->keys, ix->start, ix->rows,
                                                reinterpret_cast<const uint16_t *>(qsig), n_q, max_out, out_rows, out_count);
    else
        lsh_query_kernel<<<blocks, 256, 0, s>>>(reinterpret_cast<const uint8_t *>(ix->sig), ix->k, ix->K, ix->L,
                                                ix->cap_log2, ix->keys, ix->start, ix->rows,
                                                reinterpret_cast<const uint8_t *>(qsig), n_q, max_out, out_rows, out_count);
    WMH_LAUNCH_CHECK("lsh query");
    return WMH_OK;
}
