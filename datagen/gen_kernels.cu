// gen_kernels.cu -- device twin of datagen's counter-based generators (c1, c5).
//
// Input generation only (bench / test infrastructure, not the product): every
// entry is a pure function of (data_seed, row, col) through MurmurHash3's
// fmix64 -- integer-only, so the device and numpy (datagen/__init__.py) agree
// bit for bit.  Holds none of the method's arithmetic.
#include <cuda_runtime.h>
#include <stdint.h>

__device__ __forceinline__ uint64_t fmix64(uint64_t h) {
    h ^= h >> 33;
    h *= 0xFF51AFD7ED558CCDull;
    h ^= h >> 33;
    h *= 0xC4CEB9FE1A85EC53ull;
    h ^= h >> 33;
    return h;
}

// kind 1 (c1): 0 if low32 < z_thresh else 1 + hi32 % 15.
// kind 5 (c5): 0 if bit 63 set else #{v in 0..254 : u63 < thresh[v]} (thresh strictly decreasing).
__global__ void gen_counter_kernel(int kind, uint64_t base, int64_t row0, int64_t n_rows, int64_t dim,
                                   uint32_t z_thresh, const uint64_t *__restrict__ thresh, uint8_t *__restrict__ out) {
    __shared__ uint64_t st[256];
    if (kind == 5)
        for (int i = threadIdx.x; i < 255; i += blockDim.x) st[i] = thresh[i];
    __syncthreads();
    const int64_t total = n_rows * dim;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t n = i / dim, c = i - n * dim;
        const uint64_t b = fmix64(base ^ (uint64_t)((row0 + n) * dim + c));
        uint8_t v;
        if (kind == 1) {
            v = ((uint32_t)b < z_thresh) ? 0 : (uint8_t)(1 + (uint32_t)(b >> 32) % 15u);
        } else {
            if (b >> 63) {
                v = 0;
            } else {
                const uint64_t u = b & ((1ull << 63) - 1);
                int lo = 0, hi = 255;          // count of leading thresholds > u
                while (lo < hi) {
                    int mid = (lo + hi) >> 1;
                    if (u < st[mid]) lo = mid + 1;
                    else hi = mid;
                }
                v = (uint8_t)lo;
            }
        }
        out[i] = v;
    }
}

extern "C" int wmhgen_counter_rows(int kind, uint64_t base_mixed, int64_t row0, int64_t n_rows, int64_t dim,
                                   uint32_t z_thresh, const uint64_t *thresh_dev, uint8_t *out, void *stream) {
    if ((kind != 1 && kind != 5) || n_rows < 0 || dim < 1 || !out || (kind == 5 && !thresh_dev)) return 1;
    if (n_rows == 0) return 0;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    gen_counter_kernel<<<sms * 8, 256, 0, (cudaStream_t)stream>>>(kind, base_mixed, row0, n_rows, dim, z_thresh,
                                                                   thresh_dev, out);
    return cudaGetLastError() == cudaSuccess ? 0 : 2;
}
