// common.cuh -- internal declarations shared by the libwmh.so translation units.
// Product code (CUDA path).  Shares nothing with oracle/.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "wmh.h"

struct wmh_layout {
    int64_t dim = 0;
    uint64_t M = 0;
    uint32_t flags = 0;          // bit 0: uniform bounds
    uint32_t uniform_m = 0;      // the common bound when uniform, else 0
    uint32_t max_bound = 0;      // max_c m_c
    uint64_t digest = 0;         // FNV-1a over (dim, bounds): wmh_layout_digest
    uint32_t *bounds = nullptr;       // [dim]
    uint32_t *comp_to_m = nullptr;    // [dim + 1]   CompToM, exclusive prefix (Eq. 3)
    uint32_t *int_to_comp = nullptr;  // [M]         IntToComp (Alg. 4)
    uint32_t *cell_pack = nullptr;    // [M]         (c << 8) | (t - CompToM[c]): Alg. 5 in one load (not wide)
    uint64_t rowsum_q = 0;            // 0.1% quantile (power of two) of prepare's nonzero row sums; 0 = unknown
    double mean_s = -1.0;             // mean effective sparsity |x|_1 / M of prepare's rows (Eq. 17); < 0 = unknown
    uint64_t clamp_cells[8] = {0};    // sum_c max(0, m_c - (2^b - 1)), b = 0..7 (the plane tiles' clamp choice)
    uint64_t value_ge[8] = {0};       // sampled dense uint8 weights >= 2^b - 1 (b = 3..7; every 16th row given to prepare)
    uint64_t value_cells = 0;         // cells in that sample (0: no sample -> the bit-sliced tile clamps only to fit)
    int device = 0;
};

#define WMH_LAYOUT_UNIFORM 1u
#define WMH_LAYOUT_WIDE 2u          // some bound > 255: no cell_pack, uint16 offsets

// Device-side bounds checks of the debug library (WMH_LIB=debug, -DWMH_DEBUG):
// an index outside its array prints and traps the kernel.  Compiled out of the
// product library.
#ifdef WMH_DEBUG
#include <stdio.h>
#define WMH_DASSERT(cond)                                                                 \
    do {                                                                                  \
        if (!(cond)) {                                                                    \
            printf("WMH_DASSERT failed %s:%d: %s (block %d thread %d)\n", __FILE__, __LINE__, \
                   #cond, (int)blockIdx.x, (int)threadIdx.x);                             \
            __trap();                                                                     \
        }                                                                                 \
    } while (0)
#else
#define WMH_DASSERT(cond) \
    do {                  \
    } while (0)
#endif

namespace wmh {

// ----------------------------------------------------------------- errors
void set_error(const char *fmt, ...);
wmh_status cuda_fail(cudaError_t e, const char *what);
#define WMH_CUDA_TRY(expr, what)                                  \
    do {                                                          \
        cudaError_t _e = (expr);                                  \
        if (_e != cudaSuccess) return ::wmh::cuda_fail(_e, what); \
    } while (0)
// Every kernel launch site is followed by WMH_LAUNCH_CHECK, which also counts
// the launch (wmh_kernel_launches()).
void count_launch(unsigned n = 1);
#define WMH_LAUNCH_CHECK(what)                   \
    do {                                         \
        ::wmh::count_launch();                   \
        WMH_CUDA_TRY(cudaGetLastError(), what);  \
    } while (0)

wmh_status check_rows(const wmh_rows *rows, bool need_data);
// Optional CUDA-event bracket around the dominant (per-row) kernel of a hash
// call (wmh_hash_opts.flags & WMH_OPT_TIME_KERNEL); read with wmh_last_kernel_ms.
void kernel_timer_begin(cudaStream_t s);
void kernel_timer_end(cudaStream_t s);
int num_sms();

// ---------------------------------------------------------------- the RNG
// Reading R6-R8: a counter-based stream.  The paper's
// "r = M x Uniform(0,1)" (Alg. 3) with a consistent seed
// becomes r_t = floor(splitmix64(S ^ (j<<32) ^ t) * M / 2^64), S =
// splitmix64(seed).  SplitMix64 is the output function of Steele, Lea &
// Flood (2014).
__host__ __device__ __forceinline__ uint64_t splitmix64(uint64_t v) {
    uint64_t z = v + 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

// floor(z * M / 2^64) for M < 2^32 as two 32x32->64 multiplies:
// z*M = zh*M*2^32 + zl*M, so the top word is (zh*M + (zl*M >> 32)) >> 32.
__device__ __forceinline__ uint32_t mulhi_range(uint64_t z, uint32_t M) {
    uint32_t zl = (uint32_t)z, zh = (uint32_t)(z >> 32);
    uint64_t lo = (uint64_t)zl * M;
    uint64_t hi = (uint64_t)zh * M + (lo >> 32);
    return (uint32_t)(hi >> 32);
}

// key_hi = hi32(S) ^ j is fixed per hash; only the low word varies with t.
__device__ __forceinline__ uint32_t draw_r(uint64_t S, uint32_t j, uint32_t t, uint32_t M) {
    uint64_t key = S ^ ((uint64_t)j << 32) ^ (uint64_t)t;
    return mulhi_range(splitmix64(key), M);
}

// ------------------------------------------------- draws shared by a tile
constexpr int T0 = 256;                 // draws per hash kept in the per-launch table

// Packed cell of draw r: (c << 8) | (r - CompToM[c]) -- Alg. 5's two lookups in
// one value (bounds <= 255).  Uniform bounds: IntToComp[r] = r / m.
__device__ __forceinline__ uint32_t cell_of(uint32_t r, const uint32_t *__restrict__ pack, uint32_t uni_m) {
    if (uni_m) {
        uint32_t c = r / uni_m;
        return (c << 8) | (r - c * uni_m);
    }
    return __ldg(pack + r);
}

__device__ __forceinline__ uint2 unpack_cell(uint32_t cell) { return make_uint2(cell >> 8, cell & 0xFFu); }

// (c, r - CompToM[c]) of cell r for any layout: the division (uniform bounds),
// the packed table (bounds <= 255), else Alg. 5's two lookups IntToComp[r],
// CompToM[c] (wide layouts).
__device__ __forceinline__ uint2 cell_lookup(uint32_t r, const uint32_t *__restrict__ pack, uint32_t uni_m,
                                             const uint32_t *__restrict__ i2c, const uint32_t *__restrict__ c2m) {
    if (uni_m) {
        const uint32_t c = r / uni_m;
        return make_uint2(c, r - c * uni_m);
    }
    if (pack) return unpack_cell(__ldg(pack + r));
    const uint32_t c = __ldg(i2c + r);
    return make_uint2(c, r - __ldg(c2m + c));
}

// Sec. 3.3's alternative to the IntToComp table ("binary search over
// CompToM"): the component c with CompToM[c] <= r < CompToM[c+1], found in
// ceil(log2 D) dependent loads of the (D+1)-entry prefix array instead of one
// load of the M-entry table.  Zero-width components (CompToM[c] = CompToM[c+1],
// reading R11) never satisfy the bracket.  The measured alternative
// (WMH_OPT_ISGREEN_BINSEARCH).
__device__ __forceinline__ uint2 cell_bsearch(uint32_t r, const uint32_t *__restrict__ c2m, uint32_t D) {
    uint32_t lo = 0, hi = D;                     // CompToM[lo] <= r < CompToM[hi] (CompToM[D] = M > r)
    while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        if (__ldg(c2m + mid) <= r) lo = mid;
        else hi = mid;
    }
    return make_uint2(lo, r - __ldg(c2m + lo));
}

// weight width of a batch (wmh_rows.weight_bytes: 0 or 1 -> 1)
inline int weight_bytes(const wmh_rows &r) { return r.weight_bytes == 2 ? 2 : 1; }

// ------------------------------------------------------------ launchers
struct HashArgs {
    const wmh_layout *L;
    wmh_rows rows;
    uint64_t S;          // splitmix64(seed)
    uint32_t k, cap;
    int sig_bytes;
    void *sig;
    unsigned long long *n_sat;   // may be null
    cudaStream_t stream;
    int chunk;           // TILED: 0 = auto, else 4/8/16/32
    uint32_t horizon;    // INDEX: draws filed per hash (0 = auto)
    int tile = 0;        // TILED dense: 0 auto, 1 byte tile, 2 bit-plane tile, 3 bit-sliced tile
    void *plan_out = nullptr;    // INDEX: optional per-row plan codes (wmh_hash_opts.plan_out)
    int *tile_used = nullptr;    // TILED dense: written with the tile that ran (1/2/3)
    bool isgreen_bsearch = false;  // WMH_OPT_ISGREEN_BINSEARCH: cells by binary search over CompToM
};

wmh_status launch_hash_simple(const HashArgs &a);
wmh_status launch_hash_tiled(const HashArgs &a, bool *handled);
wmh_status launch_hash_tiled_cm(const HashArgs &a, bool *handled);
wmh_status launch_hash_tiled_bs(const HashArgs &a, bool *handled);
wmh_status launch_hash_bitslice(const HashArgs &a, bool *handled);
bool bitslice_handles(const HashArgs &a);
bool tiled_cm_full_tile(const HashArgs &a);
wmh_status launch_hash_index(const HashArgs &a, uint32_t horizon);
uint32_t index_k_max();
bool index_feasible(const wmh_layout *L, uint32_t k, uint32_t cap, uint32_t horizon);
// The index of one call, reusable by several row batches of the same (layout,
// seed, k, cap): built on a.stream, freed stream-ordered.
constexpr int IX_MAXE = 14;
struct IxEpochs {
    int E;
    uint32_t B[IX_MAXE + 1];                   // B[0] = 0, epoch e holds t < B[e + 1]
};
struct IndexBuilt {
    uint8_t *scr = nullptr;
    uint32_t *pos = nullptr, *vals = nullptr, *colstart = nullptr;
    uint2 *table = nullptr;
    unsigned long long *ctr = nullptr;
    IxEpochs ep{};
    uint32_t T = 0;
};
wmh_status index_build(const HashArgs &a, uint32_t horizon, IndexBuilt *out);
// The coalesced build of pos (E*M + 1) and vals (sum_e k * B[e+1]) (index_build.cu).
wmh_status index_build_sorted(uint64_t S, uint32_t k, uint32_t M, const IxEpochs &ep, uint32_t *pos, uint32_t *vals,
                              cudaStream_t s);
// In-place inclusive scan of uint32 a[0..n) (sums: ceil(n / 8192) + 1 words of scratch).
wmh_status scan_u32_inplace(uint32_t *a, int64_t n, uint32_t *sums, cudaStream_t s);
wmh_status index_rows(const HashArgs &a, const IndexBuilt &ix);
void index_free(IndexBuilt &ix, cudaStream_t s);
uint32_t index_horizon(const wmh_layout *L, uint32_t k, uint32_t cap, uint32_t hint);
wmh_status launch_draw_table(uint2 *table, uint32_t k, uint64_t S, uint32_t M, const uint32_t *pack, uint32_t uni_m,
                             uint32_t cmul, cudaStream_t s, const uint32_t *i2c = nullptr, const uint32_t *c2m = nullptr);

}  // namespace wmh
