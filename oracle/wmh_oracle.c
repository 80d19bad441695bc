/*
 * wmh_oracle.c -- CPU ORACLE for rejection-sampling weighted minwise hashing
 * (Shrivastava, "Exact Weighted Minwise Hashing in Constant Time", ICML 2016,
 * arXiv 1602.08393).
 *
 * THIS IS TEST INFRASTRUCTURE, NOT PRODUCT CODE.  Only tests/, the smoke() of
 * __graft_entry__.py and bench.py's cpu_baseline / --impl reference leg may
 * load it.  It shares no code, header, table or constant generator with the
 * CUDA path under paper_1602_08393_b200/ (and neither includes the other).
 *
 * It is deliberately plain and slow: every function below is the paper's
 * definition or algorithm written out in the paper's order, with no blocking,
 * fusion, table sharing or reordering.  Citations are PAPER.md line numbers
 * ("P:n") with the section / equation / algorithm they fall in; DESIGN.md
 * lists every reading (R1..R13) taken where the paper is silent, garbled or
 * inconsistent.
 *
 * Parity status: every function here is pinned by tests/test_oracle_*.py
 * against closed forms, brute force and worked examples;
 * the specific hash VALUES are pinned only relative to the RNG reading R6-R8
 * (the paper's own generator is unspecified and replaced), whose SplitMix64
 * core is pinned by its published known answer.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>

#define ORC_OK 0
#define ORC_EINVAL -1
#define ORC_EEMPTY -2
#define ORC_EOVERFLOW -3
#define ORC_EBOUND -4
#define ORC_ENOMEM -5

/* ------------------------------------------------------------------------ */
/* RNG (reading R6-R8).  The paper draws "r = M x Uniform(0,1)"   */
/* (Alg. 3) and makes the sequence consistent across vectors by      */
/* seeding.  We replace its seed chaining with a counter-based  */
/* stream: r_t for hash j is a pure function of (seed, j, t, M).            */
/* ------------------------------------------------------------------------ */

/* SplitMix64 output function (Steele, Lea & Flood 2014) applied to v:
 * the state increment by the golden gamma followed by the two
 * xor-shift-multiply rounds and the final xor-shift, all mod 2^64. */
uint64_t oracle_splitmix64(uint64_t v)
{
    uint64_t z = v + 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

/* r_t = floor(z * M / 2^64) with z = splitmix64(splitmix64(seed) ^ (j<<32) ^ t).
 * Uniform on the integer cells {0..M-1} up to a relative bias <= M/2^64
 * (reading R8: multiply-high range reduction, no rejection). */
uint32_t oracle_draw(uint64_t seed, uint32_t j, uint32_t t, uint32_t M)
{
    uint64_t S = oracle_splitmix64(seed);
    uint64_t key = S ^ ((uint64_t)j << 32) ^ (uint64_t)t;
    uint64_t z = oracle_splitmix64(key);
    unsigned __int128 prod = (unsigned __int128)z * (unsigned __int128)M;
    return (uint32_t)(prod >> 64);
}

/* ------------------------------------------------------------------------ */
/* Preprocessing: m_i (Sec. 3.1) and Alg. 4 ComputeHashMaps*/
/* ------------------------------------------------------------------------ */

/* m_c = max_n x[n][c] -- "the upper bound on the value of component x_i in
 * the given dataset"; for integer data the ceiling is the value
 * itself (reading R13). */
void oracle_colmax_dense(const uint8_t *x, int64_t n_rows, int64_t dim, uint32_t *m_out)
{
    for (int64_t c = 0; c < dim; c++) m_out[c] = 0;
    for (int64_t n = 0; n < n_rows; n++)
        for (int64_t c = 0; c < dim; c++)
            if (x[n * dim + c] > m_out[c]) m_out[c] = x[n * dim + c];
}

void oracle_colmax_csr(const int64_t *row_ptr, const int32_t *col, const uint8_t *val,
                       int64_t n_rows, int64_t dim, uint32_t *m_out)
{
    for (int64_t c = 0; c < dim; c++) m_out[c] = 0;
    for (int64_t n = 0; n < n_rows; n++)
        for (int64_t e = row_ptr[n]; e < row_ptr[n + 1]; e++)
            if (val[e] > m_out[col[e]]) m_out[col[e]] = val[e];
}

/* M = sum_i m_i (Eq. 3).  Returns ORC_EEMPTY when M = 0 and
 * ORC_EOVERFLOW when M >= 2^32 (cells are indexed by uint32). */
int oracle_total_M(const uint32_t *m, int64_t dim, uint64_t *M_out)
{
    uint64_t M = 0;
    for (int64_t c = 0; c < dim; c++) M += m[c];
    *M_out = M;
    if (M == 0) return ORC_EEMPTY;
    if (M >= (1ULL << 32)) return ORC_EOVERFLOW;
    return ORC_OK;
}

/* Alg. 4, written out literally:
 *   index = 0, CompToM[0] = 0
 *   for i = 0 .. D-1:
 *       CompToM[i+1] = M_i + CompToM[i]      (M_i here is the bound m_i, R3)
 *       for j = 0 .. M_i - 1: IntToComp[index] = i; index++
 * CompToM has D+1 entries; CompToM[D] = M (the paper stops at D-1; we also
 * keep the end so interval i is [CompToM[i], CompToM[i+1]), reading R3/R4).
 * IntToComp has exactly M entries, cells 0..M-1 (reading R4). */
int oracle_build_layout(const uint32_t *m, int64_t dim, uint32_t *comp_to_m, uint32_t *int_to_comp)
{
    uint64_t M;
    int rc = oracle_total_M(m, dim, &M);
    if (rc != ORC_OK) return rc;
    uint64_t index = 0;
    comp_to_m[0] = 0;
    for (int64_t i = 0; i < dim; i++) {
        comp_to_m[i + 1] = m[i] + comp_to_m[i];
        for (uint32_t j = 0; j < m[i]; j++) {
            int_to_comp[index] = (uint32_t)i;
            index++;
        }
    }
    return ORC_OK;
}

/* Validation that every weight is within its bound (a weight above m_c
 * would overlap the next component's interval and break Eq. 4). */
int oracle_check_bounds_dense(const uint8_t *x, int64_t n_rows, int64_t dim, const uint32_t *m,
                              int64_t *bad_row, int64_t *bad_col)
{
    for (int64_t n = 0; n < n_rows; n++)
        for (int64_t c = 0; c < dim; c++)
            if (x[n * dim + c] > m[c]) { *bad_row = n; *bad_col = c; return ORC_EBOUND; }
    return ORC_OK;
}

/* The same for CSR rows, with the structure the method relies on: row_ptr
 * non-decreasing from 0 to nnz, columns in [0, dim) and strictly ascending
 * within a row, every value within its bound.  Returns the first offending
 * nonzero (its index; for a malformed row_ptr, the row) and why:
 * 1 column out of range, 2 columns not ascending, 3 value above its bound,
 * 4 row_ptr malformed. */
int oracle_check_bounds_csr(const int64_t *row_ptr, const int32_t *col, const uint8_t *val, int64_t n_rows,
                            int64_t dim, int64_t nnz, const uint32_t *m, int64_t *bad_index, int *why)
{
    for (int64_t n = 0; n < n_rows; n++) {
        int64_t a = row_ptr[n], b = row_ptr[n + 1];
        if (a > b || a < 0 || b > nnz || (n == 0 && a != 0) || (n == n_rows - 1 && b != nnz)) {
            *bad_index = n; *why = 4; return ORC_EINVAL;
        }
        for (int64_t e = a; e < b; e++) {
            if (col[e] < 0 || col[e] >= dim) { *bad_index = e; *why = 1; return ORC_EINVAL; }
            if (e > a && col[e - 1] >= col[e]) { *bad_index = e; *why = 2; return ORC_EINVAL; }
            if (val[e] > m[col[e]]) { *bad_index = e; *why = 3; return ORC_EBOUND; }
        }
    }
    return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* ISGREEN: Alg. 5 and the Sec. 3.3 binary search       */
/* ------------------------------------------------------------------------ */

/* Alg. 5 on an integer draw (readings R1, R2): i = IntToComp[r];
 * green iff r - CompToM[i] < x_i (strict: exactly x_i green cells). */
int oracle_is_green_o1(const uint32_t *int_to_comp, const uint32_t *comp_to_m,
                       const uint8_t *x_dense, uint32_t r)
{
    uint32_t i = int_to_comp[r];
    uint32_t Mi = comp_to_m[i];
    return (r - Mi) < (uint32_t)x_dense[i];
}

/* Sec. 3.3: binary search over the row's d green intervals
 * [CompToM[c], CompToM[c] + x_c), c ascending, which are disjoint and sorted.
 * cols must be ascending and vals > 0. */
int oracle_is_green_binsearch(const uint32_t *comp_to_m, const int32_t *cols, const uint8_t *vals,
                              int64_t d, uint32_t r)
{
    int64_t lo = 0, hi = d - 1, found = -1;
    while (lo <= hi) {                 /* last interval whose start <= r */
        int64_t mid = lo + (hi - lo) / 2;
        if (comp_to_m[cols[mid]] <= r) { found = mid; lo = mid + 1; }
        else hi = mid - 1;
    }
    if (found < 0) return 0;
    return r < comp_to_m[cols[found]] + (uint32_t)vals[found];
}

/* Eq. 4 read directly: r in x_green iff there is a component c
 * with CompToM[c] <= r < CompToM[c] + x_c.  Linear scan, no tables. */
int oracle_is_green_direct(const uint32_t *comp_to_m, const uint8_t *x_dense, int64_t dim, uint32_t r)
{
    for (int64_t c = 0; c < dim; c++)
        if (comp_to_m[c] <= r && r < comp_to_m[c] + (uint32_t)x_dense[c]) return 1;
    return 0;
}

/* ------------------------------------------------------------------------ */
/* Alg. 3 Weighted MinHash with the Definition       */
/* ------------------------------------------------------------------------ */

/* Hash value from an explicitly supplied draw sequence: the 1-based index of
 * the first green draw among draws[0..cap-1] (reading R1), or cap when none
 * of the first cap draws is green (saturation, reading R9).  Used by the
 * brute-force pins, which enumerate every sequence. */
uint32_t oracle_hash_from_draws(const uint32_t *int_to_comp, const uint32_t *comp_to_m,
                                const uint8_t *x_dense, const uint32_t *draws, uint32_t cap)
{
    for (uint32_t t = 0; t < cap; t++)
        if (oracle_is_green_o1(int_to_comp, comp_to_m, x_dense, draws[t])) return t + 1;
    return cap;
}

/* One hash of one (dense) vector: Alg. 3's while loop with the counter
 * stream of oracle_draw and the cap.  h = t+1 at the first green t < cap,
 * else cap. */
uint32_t oracle_hash_one(const uint32_t *int_to_comp, const uint32_t *comp_to_m, uint32_t M,
                         const uint8_t *x_dense, uint64_t seed, uint32_t j, uint32_t cap)
{
    for (uint32_t t = 0; t < cap; t++) {
        uint32_t r = oracle_draw(seed, j, t, M);
        if (oracle_is_green_o1(int_to_comp, comp_to_m, x_dense, r)) return t + 1;
    }
    return cap;
}

typedef struct {
    int kind;                   /* 0 dense, 1 csr */
    const uint8_t *x;           /* dense */
    const int64_t *row_ptr;     /* csr */
    const int32_t *col;
    const uint8_t *val;
    int64_t n_rows, dim;
    const uint32_t *int_to_comp, *comp_to_m;
    uint32_t M;
    uint64_t seed;
    uint32_t k, cap;
    uint32_t *sig;              /* n_rows x k, row-major, h values */
    int64_t row_begin, row_end;
    int status;
} oracle_job;

static void *oracle_hash_worker(void *arg)
{
    oracle_job *jb = (oracle_job *)arg;
    uint8_t *scratch = NULL;
    if (jb->kind == 1) {
        scratch = (uint8_t *)calloc((size_t)jb->dim, 1);
        if (!scratch) { jb->status = ORC_ENOMEM; return NULL; }
    }
    for (int64_t n = jb->row_begin; n < jb->row_end; n++) {
        const uint8_t *xrow;
        if (jb->kind == 0) {
            xrow = jb->x + n * jb->dim;
        } else {                 /* scatter the CSR slice into a dense scratch row */
            for (int64_t e = jb->row_ptr[n]; e < jb->row_ptr[n + 1]; e++) scratch[jb->col[e]] = jb->val[e];
            xrow = scratch;
        }
        for (uint32_t j = 0; j < jb->k; j++)      /* Alg. 3: for i = 1 to k */
            jb->sig[n * (int64_t)jb->k + j] =
                oracle_hash_one(jb->int_to_comp, jb->comp_to_m, jb->M, xrow, jb->seed, j, jb->cap);
        if (jb->kind == 1)
            for (int64_t e = jb->row_ptr[n]; e < jb->row_ptr[n + 1]; e++) scratch[jb->col[e]] = 0;
    }
    free(scratch);
    jb->status = ORC_OK;
    return NULL;
}

/* Hash every row: sig[n][j] = h_j(x_n).  Rows are split into contiguous
 * blocks over n_threads plain pthreads (the per-row computation is
 * unchanged; threads only run different rows). */
static int oracle_hash_rows(oracle_job proto, int n_threads)
{
    if (proto.k == 0 || proto.cap == 0) return ORC_EINVAL;
    if (n_threads < 1) n_threads = 1;
    if (n_threads > proto.n_rows && proto.n_rows > 0) n_threads = (int)proto.n_rows;
    if (proto.n_rows == 0) return ORC_OK;
    oracle_job *jobs = (oracle_job *)calloc((size_t)n_threads, sizeof(oracle_job));
    pthread_t *th = (pthread_t *)calloc((size_t)n_threads, sizeof(pthread_t));
    if (!jobs || !th) { free(jobs); free(th); return ORC_ENOMEM; }
    int64_t per = (proto.n_rows + n_threads - 1) / n_threads;
    for (int i = 0; i < n_threads; i++) {
        jobs[i] = proto;
        jobs[i].row_begin = i * per;
        jobs[i].row_end = (i + 1) * per < proto.n_rows ? (i + 1) * per : proto.n_rows;
        if (jobs[i].row_begin > jobs[i].row_end) jobs[i].row_begin = jobs[i].row_end;
        pthread_create(&th[i], NULL, oracle_hash_worker, &jobs[i]);
    }
    int rc = ORC_OK;
    for (int i = 0; i < n_threads; i++) {
        pthread_join(th[i], NULL);
        if (jobs[i].status != ORC_OK) rc = jobs[i].status;
    }
    free(jobs);
    free(th);
    return rc;
}

int oracle_hash_dense(const uint8_t *x, int64_t n_rows, int64_t dim,
                      const uint32_t *int_to_comp, const uint32_t *comp_to_m, uint32_t M,
                      uint64_t seed, uint32_t k, uint32_t cap, uint32_t *sig, int n_threads)
{
    oracle_job p;
    memset(&p, 0, sizeof p);
    p.kind = 0; p.x = x; p.n_rows = n_rows; p.dim = dim;
    p.int_to_comp = int_to_comp; p.comp_to_m = comp_to_m; p.M = M;
    p.seed = seed; p.k = k; p.cap = cap; p.sig = sig;
    return oracle_hash_rows(p, n_threads);
}

int oracle_hash_csr(const int64_t *row_ptr, const int32_t *col, const uint8_t *val,
                    int64_t n_rows, int64_t dim,
                    const uint32_t *int_to_comp, const uint32_t *comp_to_m, uint32_t M,
                    uint64_t seed, uint32_t k, uint32_t cap, uint32_t *sig, int n_threads)
{
    oracle_job p;
    memset(&p, 0, sizeof p);
    p.kind = 1; p.row_ptr = row_ptr; p.col = col; p.val = val; p.n_rows = n_rows; p.dim = dim;
    p.int_to_comp = int_to_comp; p.comp_to_m = comp_to_m; p.M = M;
    p.seed = seed; p.k = k; p.cap = cap; p.sig = sig;
    return oracle_hash_rows(p, n_threads);
}

/* ------------------------------------------------------------------------ */
/* Estimation: Eq. 14-15 and the generalised Jaccard Eq. 1       */
/* ------------------------------------------------------------------------ */

/* matches_p = #{j : sig[a_p][j] == sig[b_p][j]}; J-hat = matches / k. */
void oracle_collide(const uint32_t *sig, uint32_t k, const int64_t *pairs, int64_t n_pairs,
                    uint32_t *matches)
{
    for (int64_t p = 0; p < n_pairs; p++) {
        const uint32_t *a = sig + pairs[2 * p] * (int64_t)k;
        const uint32_t *b = sig + pairs[2 * p + 1] * (int64_t)k;
        uint32_t cnt = 0;
        for (uint32_t j = 0; j < k; j++)
            if (a[j] == b[j]) cnt++;
        matches[p] = cnt;
    }
}

/* Eq. 1: J(x,y) = sum_i min(x_i,y_i) / sum_i max(x_i,y_i),
 * returned as the exact integer numerator and denominator. */
void oracle_jaccard_dense(const uint8_t *x, const uint8_t *y, int64_t dim, uint64_t *num, uint64_t *den)
{
    uint64_t mn = 0, mx = 0;
    for (int64_t c = 0; c < dim; c++) {
        mn += x[c] < y[c] ? x[c] : y[c];
        mx += x[c] > y[c] ? x[c] : y[c];
    }
    *num = mn;
    *den = mx;
}

/* Same, for two rows of a CSR matrix (columns ascending). */
void oracle_jaccard_csr(const int64_t *row_ptr, const int32_t *col, const uint8_t *val,
                        int64_t a, int64_t b, uint64_t *num, uint64_t *den)
{
    uint64_t mn = 0, mx = 0;
    int64_t i = row_ptr[a], ie = row_ptr[a + 1], k = row_ptr[b], ke = row_ptr[b + 1];
    while (i < ie || k < ke) {
        if (k >= ke || (i < ie && col[i] < col[k])) { mx += val[i]; i++; }
        else if (i >= ie || col[k] < col[i]) { mx += val[k]; k++; }
        else {
            mn += val[i] < val[k] ? val[i] : val[k];
            mx += val[i] > val[k] ? val[i] : val[k];
            i++; k++;
        }
    }
    *num = mn;
    *den = mx;
}

/* ------------------------------------------------------------------------ */
/* f1: uint16 weights (fixed-point real data, Sec. 3.1 P:137 and Sec. 4      */
/* P:322-324).  The same definitions as above with x_c in {0..65535} and    */
/* bounds m_c <= 65535; written out again (not shared with the uint8 code)   */
/* so that each can be read against the paper on its own.                    */
/* ------------------------------------------------------------------------ */

void oracle_colmax_dense16(const uint16_t *x, int64_t n_rows, int64_t dim, uint32_t *m_out)
{
    for (int64_t c = 0; c < dim; c++) m_out[c] = 0;
    for (int64_t n = 0; n < n_rows; n++)
        for (int64_t c = 0; c < dim; c++)
            if (x[n * dim + c] > m_out[c]) m_out[c] = x[n * dim + c];
}

void oracle_colmax_csr16(const int64_t *row_ptr, const int32_t *col, const uint16_t *val,
                         int64_t n_rows, int64_t dim, uint32_t *m_out)
{
    for (int64_t c = 0; c < dim; c++) m_out[c] = 0;
    for (int64_t n = 0; n < n_rows; n++)
        for (int64_t e = row_ptr[n]; e < row_ptr[n + 1]; e++)
            if (val[e] > m_out[col[e]]) m_out[col[e]] = val[e];
}

/* Alg. 5 with a uint16 weight: green iff r - CompToM[i] < x_i. */
static int oracle_is_green_o1_16(const uint32_t *int_to_comp, const uint32_t *comp_to_m,
                                 const uint16_t *x_dense, uint32_t r)
{
    uint32_t i = int_to_comp[r];
    return (r - comp_to_m[i]) < (uint32_t)x_dense[i];
}

/* Alg. 3 for one (vector, hash j) with uint16 weights. */
uint32_t oracle_hash_one16(const uint32_t *int_to_comp, const uint32_t *comp_to_m, uint32_t M,
                           const uint16_t *x_dense, uint64_t seed, uint32_t j, uint32_t cap)
{
    for (uint32_t t = 0; t < cap; t++) {
        uint32_t r = oracle_draw(seed, j, t, M);
        if (oracle_is_green_o1_16(int_to_comp, comp_to_m, x_dense, r)) return t + 1;
    }
    return cap;
}

typedef struct {
    int kind;
    const uint16_t *x;
    const int64_t *row_ptr;
    const int32_t *col;
    const uint16_t *val;
    int64_t n_rows, dim;
    const uint32_t *int_to_comp, *comp_to_m;
    uint32_t M;
    uint64_t seed;
    uint32_t k, cap;
    uint32_t *sig;
    int64_t row_begin, row_end;
    int status;
} oracle_job16;

static void *oracle_hash_worker16(void *arg)
{
    oracle_job16 *jb = (oracle_job16 *)arg;
    uint16_t *scratch = NULL;
    if (jb->kind == 1) {
        scratch = (uint16_t *)calloc((size_t)jb->dim, sizeof(uint16_t));
        if (!scratch) { jb->status = ORC_ENOMEM; return NULL; }
    }
    for (int64_t n = jb->row_begin; n < jb->row_end; n++) {
        const uint16_t *xrow;
        if (jb->kind == 0) {
            xrow = jb->x + n * jb->dim;
        } else {
            for (int64_t e = jb->row_ptr[n]; e < jb->row_ptr[n + 1]; e++) scratch[jb->col[e]] = jb->val[e];
            xrow = scratch;
        }
        for (uint32_t j = 0; j < jb->k; j++)
            jb->sig[n * (int64_t)jb->k + j] =
                oracle_hash_one16(jb->int_to_comp, jb->comp_to_m, jb->M, xrow, jb->seed, j, jb->cap);
        if (jb->kind == 1)
            for (int64_t e = jb->row_ptr[n]; e < jb->row_ptr[n + 1]; e++) scratch[jb->col[e]] = 0;
    }
    free(scratch);
    jb->status = ORC_OK;
    return NULL;
}

static int oracle_hash_rows16(oracle_job16 proto, int n_threads)
{
    if (proto.k == 0 || proto.cap == 0) return ORC_EINVAL;
    if (n_threads < 1) n_threads = 1;
    if (n_threads > proto.n_rows && proto.n_rows > 0) n_threads = (int)proto.n_rows;
    if (proto.n_rows == 0) return ORC_OK;
    oracle_job16 *jobs = (oracle_job16 *)calloc((size_t)n_threads, sizeof(oracle_job16));
    pthread_t *th = (pthread_t *)calloc((size_t)n_threads, sizeof(pthread_t));
    if (!jobs || !th) { free(jobs); free(th); return ORC_ENOMEM; }
    int64_t per = (proto.n_rows + n_threads - 1) / n_threads;
    for (int i = 0; i < n_threads; i++) {
        jobs[i] = proto;
        jobs[i].row_begin = i * per;
        jobs[i].row_end = (i + 1) * per < proto.n_rows ? (i + 1) * per : proto.n_rows;
        if (jobs[i].row_begin > jobs[i].row_end) jobs[i].row_begin = jobs[i].row_end;
        pthread_create(&th[i], NULL, oracle_hash_worker16, &jobs[i]);
    }
    int rc = ORC_OK;
    for (int i = 0; i < n_threads; i++) {
        pthread_join(th[i], NULL);
        if (jobs[i].status != ORC_OK) rc = jobs[i].status;
    }
    free(jobs);
    free(th);
    return rc;
}

int oracle_hash_dense16(const uint16_t *x, int64_t n_rows, int64_t dim,
                        const uint32_t *int_to_comp, const uint32_t *comp_to_m, uint32_t M,
                        uint64_t seed, uint32_t k, uint32_t cap, uint32_t *sig, int n_threads)
{
    oracle_job16 p;
    memset(&p, 0, sizeof p);
    p.kind = 0; p.x = x; p.n_rows = n_rows; p.dim = dim;
    p.int_to_comp = int_to_comp; p.comp_to_m = comp_to_m; p.M = M;
    p.seed = seed; p.k = k; p.cap = cap; p.sig = sig;
    return oracle_hash_rows16(p, n_threads);
}

int oracle_hash_csr16(const int64_t *row_ptr, const int32_t *col, const uint16_t *val,
                      int64_t n_rows, int64_t dim,
                      const uint32_t *int_to_comp, const uint32_t *comp_to_m, uint32_t M,
                      uint64_t seed, uint32_t k, uint32_t cap, uint32_t *sig, int n_threads)
{
    oracle_job16 p;
    memset(&p, 0, sizeof p);
    p.kind = 1; p.row_ptr = row_ptr; p.col = col; p.val = val; p.n_rows = n_rows; p.dim = dim;
    p.int_to_comp = int_to_comp; p.comp_to_m = comp_to_m; p.M = M;
    p.seed = seed; p.k = k; p.cap = cap; p.sig = sig;
    return oracle_hash_rows16(p, n_threads);
}
