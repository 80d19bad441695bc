// quantize.cu -- f1: real-valued weights in fixed point.
//
// The paper handles real x with integer bounds m_i = ceil(max) (Sec. 3.1)
// and scales the data by alpha to maximise the effective sparsity
// s = sum alpha x / sum ceil(alpha m) (Sec. 4).  On integer cells the
// exact analogue is fixed point: w = floor(x * scale) with scale = alpha * 2^f,
// hashed by the integer method with bounds max_n w (uint16 weights, "wide"
// layouts).  Scaling integer data by 2^f leaves every signature unchanged
// (r' >> f = r and r' - 2^f lo < 2^f x  <=>  r - lo < x), which is the exact
// form of P:324's "scaling up does not matter".
#include <math.h>

#include <algorithm>

#include "common.cuh"

namespace wmh {

__global__ void quantize_kernel(const float *__restrict__ in, int64_t n, float scale, uint16_t *__restrict__ out,
                                unsigned long long *__restrict__ n_bad) {
    unsigned bad = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const float x = __ldg(in + i);
        if (!(x >= 0.f)) {                       // negative or NaN: not a weight (x_i >= 0)
            bad++;
            out[i] = 0;
            continue;
        }
        const float q = floorf(__fmul_rn(x, scale));
        out[i] = q >= 65535.f ? (uint16_t)65535 : (uint16_t)q;
    }
    for (int o = 16; o; o >>= 1) bad += __shfl_xor_sync(0xFFFFFFFFu, bad, o);
    if ((threadIdx.x & 31) == 0 && bad) atomicAdd(n_bad, (unsigned long long)bad);
}

// For every scale a: num[a] += floor(x * s_a) and colmax[a][c] = max floor(x * s_a).
__global__ void scale_objective_kernel(const float *__restrict__ x, const int32_t *__restrict__ col, int64_t n,
                                       int64_t dim, const float *__restrict__ scales, int n_scales,
                                       uint32_t *__restrict__ colmax, unsigned long long *__restrict__ num,
                                       unsigned long long *__restrict__ clipped) {
    for (int a = 0; a < n_scales; a++) {
        const float sc = scales[a];
        unsigned long long acc = 0;
        unsigned clip = 0;
        for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
            const float v = __ldg(x + i);
            if (!(v > 0.f)) continue;
            const float qf = floorf(__fmul_rn(v, sc));
            const uint32_t q = qf >= 65535.f ? 65535u : (uint32_t)qf;
            clip += qf >= 65536.f;
            acc += q;
            const int64_t c = col ? (int64_t)__ldg(col + i) : i % dim;
            uint32_t *dst = colmax + (int64_t)a * dim + c;
            if (q > *((volatile uint32_t *)dst)) atomicMax(dst, q);
        }
        for (int o = 16; o; o >>= 1) {
            acc += __shfl_xor_sync(0xFFFFFFFFu, acc, o);
            clip += __shfl_xor_sync(0xFFFFFFFFu, clip, o);
        }
        if ((threadIdx.x & 31) == 0 && acc) atomicAdd(num + a, acc);
        if ((threadIdx.x & 31) == 0 && clip) atomicAdd(clipped + a, (unsigned long long)clip);
    }
}

__global__ void sum_rows_kernel(const uint32_t *__restrict__ colmax, int64_t dim, unsigned long long *__restrict__ den) {
    const int a = blockIdx.y;
    unsigned long long acc = 0;
    for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < dim; c += (int64_t)gridDim.x * blockDim.x)
        acc += colmax[(int64_t)a * dim + c];
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xFFFFFFFFu, acc, o);
    if ((threadIdx.x & 31) == 0 && acc) atomicAdd(den + a, acc);
}

}  // namespace wmh

using namespace wmh;

extern "C" wmh_status wmh_quantize(const float *in, int64_t n, float scale, uint16_t *out, void *stream) {
    if (n < 0) { set_error("wmh_quantize: n < 0"); return WMH_EINVAL; }
    if (!(scale > 0.f) || !isfinite(scale)) { set_error("wmh_quantize: scale must be finite and > 0"); return WMH_EINVAL; }
    if (n == 0) return WMH_OK;
    if (!in || !out) { set_error("wmh_quantize: NULL pointer"); return WMH_EINVAL; }
    cudaStream_t s = (cudaStream_t)stream;
    unsigned long long *bad = nullptr, hb = 0;
    WMH_CUDA_TRY(cudaMallocAsync((void **)&bad, sizeof hb, s), "quantize scratch");
    WMH_CUDA_TRY(cudaMemsetAsync(bad, 0, sizeof hb, s), "quantize scratch memset");
    const int64_t blocks = std::min<int64_t>((int64_t)num_sms() * 16, (n + 255) / 256);
    quantize_kernel<<<(unsigned)blocks, 256, 0, s>>>(in, n, scale, out, bad);
    WMH_LAUNCH_CHECK("quantize launch");
    cudaError_t e1 = cudaMemcpyAsync(&hb, bad, sizeof hb, cudaMemcpyDeviceToHost, s);
    cudaError_t e2 = cudaStreamSynchronize(s);
    cudaFreeAsync(bad, s);
    if (e1 != cudaSuccess || e2 != cudaSuccess) return cuda_fail(e1 != cudaSuccess ? e1 : e2, "quantize readback");
    if (hb) { set_error("wmh_quantize: %llu weights are negative or NaN", hb); return WMH_EINVAL; }
    return WMH_OK;
}

extern "C" wmh_status wmh_scale_objective(const wmh_rows *rows, const float *scales, int32_t n_scales, uint64_t *out,
                                          void *stream) {
    if (!rows || !scales || !out) { set_error("wmh_scale_objective: NULL pointer"); return WMH_EINVAL; }
    if (n_scales < 1 || n_scales > 1024) { set_error("wmh_scale_objective: n_scales=%d not in [1, 1024]", (int)n_scales); return WMH_EINVAL; }
    wmh_rows r = *rows;
    r.weight_bytes = 1;                          // float data: structure checks only
    wmh_status st = check_rows(&r, true);
    if (st != WMH_OK) return st;
    for (int a = 0; a < n_scales; a++)
        if (!(scales[a] > 0.f) || !isfinite(scales[a])) { set_error("wmh_scale_objective: scale %d not finite > 0", a); return WMH_EINVAL; }
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t dim = rows->dim;
    const int64_t n = rows->kind == WMH_DENSE ? rows->n_rows * dim : rows->nnz;
    const size_t cm_bytes = sizeof(uint32_t) * (size_t)dim * n_scales;
    uint8_t *scr = nullptr;
    WMH_CUDA_TRY(cudaMallocAsync((void **)&scr, cm_bytes + 24 * (size_t)n_scales + 4 * (size_t)n_scales + 256, s),
                 "scale objective scratch");
    uint32_t *colmax = reinterpret_cast<uint32_t *>(scr);
    unsigned long long *num = reinterpret_cast<unsigned long long *>(scr + ((cm_bytes + 15) & ~(size_t)15));
    unsigned long long *den = num + n_scales;
    unsigned long long *clipped = den + n_scales;
    float *dsc = reinterpret_cast<float *>(clipped + n_scales);
    st = WMH_OK;
    do {
        if (cudaMemsetAsync(scr, 0, ((cm_bytes + 15) & ~(size_t)15) + 24 * (size_t)n_scales, s) != cudaSuccess ||
            cudaMemcpyAsync(dsc, scales, sizeof(float) * n_scales, cudaMemcpyHostToDevice, s) != cudaSuccess) {
            st = cuda_fail(cudaGetLastError(), "scale objective setup");
            break;
        }
        if (n > 0) {
            const int64_t blocks = std::min<int64_t>((int64_t)num_sms() * 8, (n + 255) / 256);
            scale_objective_kernel<<<(unsigned)blocks, 256, 0, s>>>(
                reinterpret_cast<const float *>(rows->kind == WMH_DENSE ? rows->dense : rows->val),
                rows->kind == WMH_DENSE ? nullptr : rows->col, n, dim, dsc, n_scales, colmax, num, clipped);
            count_launch();
            const int64_t bx = std::min<int64_t>(64, (dim + 255) / 256);
            sum_rows_kernel<<<dim3((unsigned)bx, (unsigned)n_scales), 256, 0, s>>>(colmax, dim, den);
            count_launch();
            if (cudaGetLastError() != cudaSuccess) { st = cuda_fail(cudaGetLastError(), "scale objective launch"); break; }
        }
        unsigned long long h[3072];
        cudaError_t e1 = cudaMemcpyAsync(h, num, 24 * (size_t)n_scales, cudaMemcpyDeviceToHost, s);
        cudaError_t e2 = cudaStreamSynchronize(s);
        if (e1 != cudaSuccess || e2 != cudaSuccess) { st = cuda_fail(e1 != cudaSuccess ? e1 : e2, "scale objective readback"); break; }
        for (int a = 0; a < n_scales; a++) {
            out[3 * a] = h[a];
            out[3 * a + 1] = h[n_scales + a] * (uint64_t)rows->n_rows;
            out[3 * a + 2] = h[2 * n_scales + a];
        }
    } while (0);
    cudaFreeAsync(scr, s);
    return st;
}

// Sec. 4's alpha = arg max sum(alpha x) / sum(ceil(alpha m)) over the
// candidate grid, evaluated with wmh_scale_objective: among the scales that do
// not saturate a uint16 weight, the largest mean effective sparsity
// num / den (compared exactly as num_a * den_b > num_b * den_a in 128 bits);
// ties go to the smaller scale (the smaller M; reading R18).
extern "C" wmh_status wmh_choose_scale(const wmh_rows *rows, const float *scales, int32_t n_scales, int32_t *best,
                                       void *stream) {
    if (!best) { set_error("wmh_choose_scale: best is NULL"); return WMH_EINVAL; }
    *best = -1;
    if (n_scales < 1 || n_scales > 1024) { set_error("wmh_choose_scale: n_scales=%d not in [1, 1024]", (int)n_scales); return WMH_EINVAL; }
    uint64_t obj[3 * 1024];
    wmh_status st = wmh_scale_objective(rows, scales, n_scales, obj, stream);
    if (st != WMH_OK) return st;
    int b = -1;
    for (int a = 0; a < n_scales; a++) {
        const uint64_t num = obj[3 * a], den = obj[3 * a + 1], clipped = obj[3 * a + 2];
        if (den == 0 || clipped) continue;
        if (b < 0) { b = a; continue; }
        const unsigned __int128 lhs = (unsigned __int128)num * obj[3 * b + 1], rhs = (unsigned __int128)obj[3 * b] * den;
        if (lhs > rhs || (lhs == rhs && scales[a] < scales[b])) b = a;
    }
    if (b < 0) { set_error("wmh_choose_scale: every candidate scale quantises the rows to zero or saturates a weight"); return WMH_EINVAL; }
    *best = b;
    return WMH_OK;
}
