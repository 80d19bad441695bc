/*
 * wmh.h -- C ABI of libwmh.so: B200 (sm_100a) rejection-sampling weighted
 * minwise hashing (Shrivastava, "Exact Weighted Minwise Hashing in Constant
 * Time", ICML 2016, arXiv 1602.08393).
 *
 * Citations are PAPER.md line numbers "P:n" with the section / equation /
 * algorithm they fall in; readings R1..R16 are listed in DESIGN.md §2.
 *
 * Conventions shared by every entry point
 * ---------------------------------------
 *  - Plain C types only.  Every array argument is a DEVICE pointer owned by
 *    the caller (typically a torch tensor) unless the name says _host.  The
 *    library never frees caller memory.
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default
 *    stream).  Calls are asynchronous and stream-ordered; the only
 *    host<->device synchronisations are the ones a function documents.
 *  - Every call returns a wmh_status.  On failure a human-readable message is
 *    available from wmh_last_error() (thread-local, valid until the next
 *    call on the same thread).  Arguments are validated before any launch;
 *    an invalid call launches nothing and leaves outputs untouched.
 *  - Weights are integers: uint8 (x in {0..255}) or uint16 (x in {0..65535},
 *    wmh_rows.weight_bytes = 2).  The paper quantises to integer bounds
 *    m_i = ceil(max) (Sec. 3.1); real-valued inputs are scaled and
 *    quantised to uint16 fixed point by wmh_quantize (Sec. 4).
 *  - There is no CPU fallback: without a CUDA device every compute call
 *    fails with WMH_ECUDA.
 */
#ifndef WMH_H
#define WMH_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    WMH_OK = 0,
    WMH_EINVAL = 1,    /* an argument is out of its documented domain            */
    WMH_EBOUND = 2,    /* a weight exceeds its bound m_c (row, col in last_error) */
    WMH_EEMPTY = 3,    /* M = sum m_c = 0: no cell exists to draw from            */
    WMH_EOVERFLOW = 4, /* M >= 2^32: cells are indexed by uint32                  */
    WMH_ECUDA = 5,     /* CUDA runtime / launch failure (or no device)            */
    WMH_ENOMEM = 6     /* device allocation failed                                */
} wmh_status;

typedef enum { WMH_DENSE = 0, WMH_CSR = 1 } wmh_kind;

/* A batch of non-negative integer vectors x (Sec. 2: "x_i >= 0").
 *  kind = WMH_DENSE: `dense` is n_rows x dim uint8, row-major, row n at
 *                    dense + n*dim.  row_ptr/col/val are ignored.
 *  kind = WMH_CSR:   row_ptr (int64, n_rows+1, row_ptr[0] = 0,
 *                    non-decreasing), col (int32, nnz, strictly ascending
 *                    within a row, 0 <= col < dim), val (uint8, nnz, > 0);
 *                    nnz must equal row_ptr[n_rows] (host copy of it, so the
 *                    library need not read it back).  Explicit zeros are
 *                    allowed but wasteful.
 * n_rows may be 0 (every call is then a no-op returning WMH_OK). */
typedef struct {
    int32_t kind;
    int64_t n_rows;
    int64_t dim;
    const uint8_t *dense;
    const int64_t *row_ptr;
    const int32_t *col;
    const uint8_t *val;
    int64_t nnz;
    int32_t weight_bytes;  /* 1 (uint8 weights; 0 also means 1) or 2: `dense` / `val`
                              then point to uint16 weights (cast), for fixed-point
                              real-valued data (P:137 ceil bound, Sec. 4 scaling;
                              see wmh_quantize).  Bounds may then reach 65535. */
} wmh_rows;

/* Opaque, immutable red-green layout (Eq. 4; Alg. 4).
 * Owned by the library; share it read-only across streams and threads;
 * free it with wmh_layout_free after all work using it has completed. */
typedef struct wmh_layout wmh_layout;

/* ---- a1: column maxima --------------------------------------------------
 * colmax[c] = max_n x[n][c] over the given rows (the per-coordinate bound m_i
 * "computed (estimated) while reading the data").
 * colmax: device uint32[dim], fully overwritten.  Multi-GPU callers reduce
 * the per-rank results with an all-reduce(MAX) / all-gather + max before
 * wmh_prepare so that M, and hence every draw, is identical on every rank
 * (the random sequence must be consistent across vectors).
 * Errors: EINVAL (null pointers, dim < 1, n_rows < 0, bad kind), ECUDA. */
wmh_status wmh_colmax(const wmh_rows *rows, uint32_t *colmax, void *stream);

/* ---- f1: real-valued weights in fixed point (Sec. 3.1, Sec. 4)
 * out[i] = min(65535, floor(in[i] * scale)) for n float32 weights in >= 0
 * (the product rounded to nearest in float32, then floored), so a row of reals
 * becomes the uint16 integer vector the integer method hashes exactly.  With
 * scale = alpha * 2^f the bounds are the column maxima of the quantised rows
 * (wmh_colmax), and a weight loses at most 1/scale.  Dyadic weights x = w/scale
 * with integer w <= 65535 are exact.  in/out: device, n elements.
 * Errors: EINVAL (null, n < 0, scale not finite or <= 0, a weight < 0 or NaN:
 * reported after one synchronisation of `stream`), ECUDA. */
wmh_status wmh_quantize(const float *in, int64_t n, float scale, uint16_t *out, void *stream);

/* Sec. 4's choice of the scale ("alpha = arg max sum alpha x_i /
 * sum ceil(alpha m_i)"), evaluated for fixed-point quantisation: for each
 * candidate scale s_a the numerator sum_n sum_c floor(x * s_a) and the
 * denominator n_rows * sum_c max_n floor(x * s_a) of the mean effective
 * sparsity (Eq. 17) of the quantised rows.  rows_f32 uses the wmh_rows layout
 * with FLOAT weights (dense / val point to float32, weight_bytes ignored).
 * scales: host array of n_scales (<= 1024); out: host uint64[3 * n_scales]:
 * (num, den, clipped) with clipped = #weights whose floor(x * s_a) >= 65536 (the
 * uint16 quantiser would saturate them; such a scale changes the data).
 * Synchronises `stream`.  Errors: EINVAL, ENOMEM, ECUDA. */
wmh_status wmh_scale_objective(const wmh_rows *rows_f32, const float *scales, int32_t n_scales, uint64_t *out,
                               void *stream);

/* Sec. 4's scale choice itself: *best = the index in scales[] of the
 * candidate with the largest mean effective sparsity num / den (from
 * wmh_scale_objective, compared exactly in 128-bit integers) among those that
 * saturate no uint16 weight; ties go to the smaller scale (reading R18).
 * Synchronises `stream`.  Errors: EINVAL (no admissible scale; bad arguments),
 * ENOMEM, ECUDA. */
wmh_status wmh_choose_scale(const wmh_rows *rows_f32, const float *scales, int32_t n_scales, int32_t *best,
                            void *stream);

/* ---- a3 + a4: prefix sums and Alg. 4 ComputeHashMaps --------------------
 * Builds CompToM[c] = sum_{i<c} m_i (Eq. 3; exclusive prefix, interval
 * c = [CompToM[c], CompToM[c+1]), reading R3) and IntToComp[t] = c for every
 * integer cell t of interval c (Alg. 4; M cells, reading R4).
 * Components with m_c = 0 get no cells (reading R11).
 *   bounds: device uint32[dim], every m_c <= 65535 (bounds above 255 make a
 *           "wide" layout, hashed by the INDEX and SIMPLE kernels);
 *           copied, so the caller may free it after the call returns.
 *   rows:   optional (may be NULL).  When given, every weight is checked
 *           against its bound (and CSR structure is validated); the first
 *           offender is reported as WMH_EBOUND / WMH_EINVAL.
 * Synchronises `stream` once to read back M (8 bytes) and the checks.
 * Errors: EINVAL (null, dim < 1, a bound > 65535, malformed CSR), EBOUND,
 *         EEMPTY (M = 0), EOVERFLOW (M >= 2^32), ENOMEM, ECUDA. */
wmh_status wmh_prepare(const uint32_t *bounds, int64_t dim, const wmh_rows *rows, wmh_layout **out,
                       void *stream);

/* Layout facts (host values): dim, M, flags (bit 0: every m_c equal, so
 * IntToComp is the division r / m; bit 1: "wide", some m_c > 255), the
 * uniform bound (0 if not uniform). */
wmh_status wmh_layout_info(const wmh_layout *layout, int64_t *dim, uint64_t *M, uint32_t *flags,
                           uint32_t *uniform_bound);

/* A 64-bit digest of the layout: FNV-1a over dim and the bounds m_c (host
 * value, computed once by wmh_prepare).  Signatures are comparable only when
 * made with the same (seed, k, cap) over layouts with equal digests -- equal
 * bounds give the same M, CompToM and draw stream (SPEC's
 * same-layout rule).  The Python binding carries it with each
 * Sketch and refuses to collide mismatched ones.  Errors: NULL arguments. */
wmh_status wmh_layout_digest(const wmh_layout *layout, uint64_t *digest);

/* Read-only DEVICE views of the layout's tables, for tests: comp_to_m
 * (uint32[dim+1]), int_to_comp (uint32[M]), bounds (uint32[dim]). */
wmh_status wmh_layout_tables(const wmh_layout *layout, const uint32_t **comp_to_m,
                             const uint32_t **int_to_comp, const uint32_t **bounds);

void wmh_layout_free(wmh_layout *layout);

/* Check rows against an existing layout: every weight x[n][c] <= m_c (the
 * condition Eq. 2 and Alg. 5 rely on) and, for CSR, the
 * structure (row_ptr monotone, columns ascending and < dim).  For rows that
 * wmh_prepare did not see (streaming batches, a second dataset sketched with
 * the first one's layout).  Reads the rows once (dense: one column-max pass;
 * the first offender is located only on failure) and synchronises `stream`.
 * Errors: EBOUND (first offending (row, col) / nonzero in wmh_last_error),
 *         EINVAL (null, dim mismatch, malformed CSR), ENOMEM, ECUDA. */
wmh_status wmh_check_rows(const wmh_layout *layout, const wmh_rows *rows, void *stream);

/* ---- a5..a9: the hash ------------------------------------------------------
 * sig[n][j] = h_j(x_n), j = 0..k-1, row-major n_rows x k, for every row:
 *   S   = splitmix64(seed)                                   (reading R7)
 *   r_t = floor(splitmix64(S ^ (j << 32) ^ t) * M / 2^64)     (R6, R8)
 *   c   = IntToComp[r_t];  green iff r_t - CompToM[c] < x_c  (Alg. 5, P:297-316;
 *                                                             R1, R2)
 *   h   = t + 1 for the first green t < cap, else cap         (Alg. 3, P:158-180;
 *                                                             Def.; R9)
 * Draws depend only on (seed, j, t, M) -- never on x (the consistency of
 * P:190-191) -- so rows may be sharded across GPUs freely.  An all-zero row
 * yields cap for every j (reading R12).
 *   rows must satisfy x <= bounds of `layout` (checked by wmh_prepare when
 *        given rows; not re-checked here unless wmh_hash_ex gets
 *        WMH_OPT_VALIDATE -- otherwise a weight above its bound gives
 *        signatures that are silently wrong and kernel-dependent; see
 *        wmh_check_rows) and rows->dim == layout dim.
 *   k >= 1; 1 <= cap <= 2^(8*sig_bytes) - 1; sig_bytes in {1, 2}.
 *   sig_out: device, n_rows*k*sig_bytes bytes (uint8 or uint16 values).
 *   n_saturated: optional device uint64, INCREMENTED (not overwritten) by
 *        the number of (row, j) that reached the cap without a green draw.
 * Output is bit-identical to the CPU oracle for the same inputs.
 * Errors: EINVAL, ENOMEM (scratch), ECUDA. */
wmh_status wmh_hash(const wmh_layout *layout, const wmh_rows *rows, uint64_t seed, uint32_t k, uint32_t cap,
                    int32_t sig_bytes, void *sig_out, uint64_t *n_saturated, void *stream);

/* Kernel selection for tests and benchmarks (all variants are bit-identical). */
typedef enum {
    WMH_ALGO_AUTO = 0,   /* pick per input (the default used by wmh_hash)         */
    WMH_ALGO_SIMPLE = 1, /* one thread per (row, j), global-table lookups         */
    WMH_ALGO_TILED = 2,  /* dense rows staged in shared memory, draws shared by a tile
                            (CSR rows: WMH_EINVAL "does not take this input shape") */
    WMH_ALGO_INDEX = 3   /* draws (j, t < T) filed once per call under their cell; a
                            row visits only its green draws, then Alg. 3's loop from
                            t = T for hashes still unresolved; k up to ~54,000 on
                            B200 (h[k] lives in shared memory) and a key space
                            E*M <= 5.4e8 cells (E = 1..10 nested epochs): beyond
                            either AUTO picks another kernel and an explicit
                            request gets WMH_EINVAL */
} wmh_algo;

typedef struct {
    int32_t algo;        /* wmh_algo */
    int32_t chunk;       /* TILED: draws tested per row before re-queueing it, one of
                            0 (auto: picked per tile from its effective sparsity
                            s = |x|_1 / M, Eq. 17), 4, 8, 16, 32 */
    int32_t algo_used;   /* OUTPUT: written by wmh_hash_ex with the kernel that ran (wmh_algo) */
    uint32_t horizon;    /* INDEX: draws t < horizon of every hash are filed (0 = auto:
                            from the row-sum statistics wmh_prepare gathered, else cap);
                            clamped to [1, cap].  Performance only: results do not depend
                            on it.  OUTPUT when the index kernel ran: the horizon it used */
    uint32_t flags;      /* WMH_OPT_TIME_KERNEL: bracket the call's dominant (per-row)
                            kernel with CUDA events on `stream`; read with
                            wmh_last_kernel_ms.  WMH_OPT_TILE_BYTES /
                            WMH_OPT_TILE_BITPLANES / WMH_OPT_TILE_BITSLICE
                            (exclusive): for TILED on dense rows, the byte tile,
                            the round-1 bit-plane tile or the lane-per-draw
                            bit-sliced tile (default: the bit-sliced tile when
                            its planes fit).  Performance only. */
    void *plan_out;      /* optional device uint8[n_rows] (may be NULL): when the INDEX
                            kernel runs, its per-row plan code -- bits 0-3 the epoch
                            (horizon) the row picked, bit 4 columns staged in shared
                            memory, bit 5 Alg. 3's fallback loop ran, bit 6 more
                            nonzeros than one range batch, bit 7 all-zero row.  For
                            tests that must cover every plan; results do not depend on it */
    int32_t tile_used;   /* OUTPUT: with algo_used == WMH_ALGO_TILED on dense rows, the tile
                            that ran: 1 byte tile, 2 bit-plane tile, 3 bit-sliced tile */
    int32_t reserved[3]; /* must be zero */
} wmh_hash_opts;

#define WMH_OPT_TIME_KERNEL 1u
#define WMH_OPT_TILE_BYTES 2u
#define WMH_OPT_TILE_BITPLANES 4u
#define WMH_OPT_TILE_BITSLICE 8u
#define WMH_OPT_ISGREEN_BINSEARCH 32u  /* Alg. 5's component lookup by binary search over
                                         CompToM (Sec. 3.3) instead of the IntToComp
                                         table: SIMPLE per draw, the tiles' draw tables.
                                         Same results; the measured alternative */
#define WMH_OPT_VALIDATE 16u      /* check every row against the layout's bounds first
                                     (wmh_check_rows): WMH_EBOUND instead of silently
                                     wrong signatures for x_c > m_c.  One extra pass
                                     over the rows and one synchronisation */

wmh_status wmh_hash_ex(const wmh_layout *layout, const wmh_rows *rows, uint64_t seed, uint32_t k,
                       uint32_t cap, int32_t sig_bytes, void *sig_out, uint64_t *n_saturated,
                       wmh_hash_opts *opts, void *stream);

/* A prepared hash family for streaming many row batches: wmh_hasher_create
 * draws every (j, t < T) once and files it under its cell (the INDEX kernel's
 * build, see WMH_ALGO_INDEX; horizon as in wmh_hash_opts, 0 = auto);
 * wmh_hasher_run then hashes a batch with the index kernel's row pass only.
 * Output is bit-identical to wmh_hash(layout, rows, seed, k, cap, ...).  The
 * hasher keeps a pointer to `layout` (keep it alive) and its device index
 * (freed by wmh_hasher_free, which synchronises the device).  Every run waits
 * (stream-ordered, cudaStreamWaitEvent) for the build recorded on the create
 * stream and uses a row counter of its own, so runs may be issued on any
 * streams, concurrently.  Errors: as wmh_hash; k within the index kernel's
 * limit (WMH_ALGO_INDEX). */
typedef struct wmh_hasher wmh_hasher;
wmh_status wmh_hasher_create(const wmh_layout *layout, uint64_t seed, uint32_t k, uint32_t cap, uint32_t horizon,
                             wmh_hasher **out, void *stream);
wmh_status wmh_hasher_run(const wmh_hasher *hasher, const wmh_rows *rows, int32_t sig_bytes, void *sig_out,
                          uint64_t *n_saturated, void *stream);
void wmh_hasher_free(wmh_hasher *hasher);

/* End-to-end convenience (the e2e path): rows and signatures in HOST memory
 * (pinned or pageable).  Copies the rows host->device into library scratch
 * (kept across calls and grown on demand, one per thread), runs wmh_hash on
 * `stream`, copies the signatures device->host and synchronises `stream`.
 * rows_host uses the wmh_rows layout with HOST pointers.  Errors: as wmh_hash. */
wmh_status wmh_hash_host(const wmh_layout *layout, const wmh_rows *rows_host, uint64_t seed, uint32_t k,
                         uint32_t cap, int32_t sig_bytes, void *sig_out_host, void *stream);

/* ---- a10: signature agreement (Eq. 14-15) -----------------------
 * matches[p] = #{ j : sig[a_p][j] == sig[b_p][j] } for pairs[p] = (a_p, b_p)
 * (device int64[n_pairs][2]); optional jhat[p] = matches[p] / k as an IEEE
 * round-to-nearest float (J-hat of Eq. 14).  sig is n_rows x k of sig_bytes.
 * Pair indices must lie in [0, n_rows): out-of-range pairs get matches = 0
 * and jhat = NaN, and the call returns WMH_EINVAL after synchronising
 * `stream` once to count them (only when check_pairs != 0).
 * Errors: EINVAL, ECUDA. */
wmh_status wmh_collide(const void *sig, int32_t sig_bytes, uint32_t k, int64_t n_rows, const int64_t *pairs,
                       int64_t n_pairs, uint32_t *matches, float *jhat, int32_t check_pairs, void *stream);

/* a10 across two signature buffers (e.g. a query set against a corpus, or two
 * sketches made separately with the same seed, k, cap and layout): pair p
 * compares row pairs[2p] of sig_a (n_a rows) with row pairs[2p+1] of sig_b
 * (n_b rows); both k columns wide, sig_bytes each.  Same outputs, checks and
 * errors as wmh_collide (check_pairs: indices outside [0, n_a) x [0, n_b)
 * -> WMH_EINVAL after one synchronisation). */
wmh_status wmh_collide2(const void *sig_a, int64_t n_a, const void *sig_b, int64_t n_b, int32_t sig_bytes,
                        uint32_t k, const int64_t *pairs, int64_t n_pairs, uint32_t *matches, float *jhat,
                        int32_t check_pairs, void *stream);

/* Device time (ms) of the dominant kernel of the last wmh_hash_ex call on this
 * thread that set WMH_OPT_TIME_KERNEL (CUDA events on its stream).  Waits for
 * that kernel to finish.  Errors: EINVAL (no such call), ECUDA. */
wmh_status wmh_last_kernel_ms(float *ms);

/* ---- f3: (K, L) banding LSH over the signatures ---------------------
 * Band b of a signature row is its hashes [bK, (b+1)K); a row is a candidate of
 * a query when they are equal in at least one band, which happens with
 * probability 1 - (1 - J^K)^L for a pair of generalized Jaccard J (Theorem 1).
 * wmh_lsh_build indexes the n_rows x k signatures `sig` (device, sig_bytes 1 or
 * 2, K*L <= k): per band a key of the K values, a bucket table and the rows
 * grouped by bucket (device memory owned by the index).  `sig` is NOT copied:
 * it must stay alive and unchanged while the index is used.
 * wmh_lsh_query: for each of the n_q query rows `qsig` (device, same k and
 * sig_bytes) writes out_count[q] = the number of distinct candidate rows (each
 * reported once, for its first colliding band; band values compared exactly,
 * so bucket-key collisions never add a candidate) and up to max_out of them to
 * out_rows[q][0..max_out) (device int64; which ones when there are more is
 * unspecified; unused slots untouched).  Asynchronous on `stream`.
 * Errors: EINVAL, ENOMEM, ECUDA. */
typedef struct wmh_lsh wmh_lsh;
wmh_status wmh_lsh_build(const void *sig, int32_t sig_bytes, uint32_t k, int64_t n_rows, uint32_t K, uint32_t L,
                         wmh_lsh **out, void *stream);
wmh_status wmh_lsh_query(const wmh_lsh *index, const void *qsig, int64_t n_q, uint32_t max_out, int64_t *out_rows,
                         uint32_t *out_count, void *stream);
void wmh_lsh_free(wmh_lsh *index);

/* Thread-local description of the last failure ("" if none). */
const char *wmh_last_error(void);

/* One empty kernel launched on `stream`: the launch floor against which the
 * launch-bound configuration c1 is reported (bench.py --graph).  Errors: ECUDA. */
wmh_status wmh_empty_launch(void *stream);

/* Library version string, e.g. "wmh 0.1 sm_100a". */
const char *wmh_version(void);

/* Number of CUDA kernels this library has launched in the process so far
 * (all entry points; a monotone counter for launch accounting in benchmarks). */
uint64_t wmh_kernel_launches(void);

#ifdef __cplusplus
}
#endif
#endif /* WMH_H */
