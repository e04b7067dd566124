// Operand preparation kernels: fp32 -> bf16 staging of q / kc (round to
// nearest even, with representability and finiteness flags), sentinel fill
// of running top-k buffers, the optional boolean mask tile (causal.cpp:43-79)
// and a counter-based synthetic input generator for large benchmark shapes.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.h"

namespace {

__global__ void convert_bf16_kernel(const ConvertParams p) {
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    bool inexact = false, nonfinite = false;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < p.n; i += stride) {
        const float x = p.src[i];
        const __nv_bfloat16 h = __float2bfloat16_rn(x);
        p.dst[i] = h;
        if (!isfinite(x)) nonfinite = true;
        if (__bfloat162float(h) != x) inexact = true;
    }
    if (nonfinite && p.nonfinite_flag) atomicOr(p.nonfinite_flag, 1);
    if (inexact && p.inexact_flag) atomicOr(p.inexact_flag, 1);
}

__global__ void fill_sentinel_kernel(float* val, int32_t* idx, int64_t n) {
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    const float neg_inf = -__int_as_float(0x7f800000);
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
        val[i] = neg_inf;
        idx[i] = -1;
    }
}

__global__ void bool_mask_kernel(uint8_t* keep, int64_t rows, int64_t cols, int64_t s0, int64_t t0,
                                 int64_t ratio) {
    const int64_t n = rows * cols;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < n; e += stride) {
        const int64_t i = e / cols, j = e % cols;
        keep[e] = (t0 + j < (s0 + i + 1) / ratio) ? 1 : 0;
    }
}

__global__ void apply_bool_mask_kernel(float* scores, int64_t ld, const uint8_t* keep, int64_t batch,
                                       int64_t rows, int64_t cols) {
    const int64_t n = batch * rows * cols;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    const float neg_inf = -__int_as_float(0x7f800000);
    for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < n; e += stride) {
        const int64_t j = e % cols;
        const int64_t bi = e / cols;  // b * rows + i
        const int64_t i = bi % rows;
        if (keep[i * cols + j] == 0) scores[bi * ld + j] = neg_inf;
    }
}

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

// Element e of stream (seed, sid): Box-Muller pair (e >> 1), cos for even e,
// sin for odd e, uniforms from a splitmix64 hash of the pair counter. Same
// distribution as synth.cpp:50-64, different (counter-based) stream so any
// slice can be produced independently on device.
__device__ __forceinline__ float gen_one(int64_t e, double stddev, uint64_t seed, uint64_t sid) {
    const uint64_t base = seed * 0x9E3779B97F4A7C15ULL + sid * 0xD1B54A32D192ED03ULL;
    const uint64_t pair = static_cast<uint64_t>(e >> 1);
    const uint64_t z1 = mix64(base + 2 * pair + 1);
    const uint64_t z2 = mix64(base + 2 * pair + 2 + 0x632BE59BD9B4E019ULL);
    const float u1 = static_cast<float>(((z1 >> 40) + 1)) * (1.0f / 16777216.0f);  // (0, 1]
    const float u2 = static_cast<float>(z2 >> 40) * (1.0f / 16777216.0f);          // [0, 1)
    const float r = sqrtf(-2.0f * logf(u1));
    float sv, cv;
    sincospif(2.0f * u2, &sv, &cv);
    return static_cast<float>(((e & 1) ? sv : cv) * r * static_cast<float>(stddev));
}

__global__ void gen_bf16_kernel(__nv_bfloat16* dst, int64_t n, double stddev, uint64_t seed, uint64_t sid,
                                int64_t offset) {
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
        dst[i] = __float2bfloat16_rn(gen_one(offset + i, stddev, seed, sid));
    }
}

__global__ void gen_f32_kernel(float* dst, int64_t n, double stddev, uint64_t seed, uint64_t sid,
                               int64_t offset) {
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
        dst[i] = gen_one(offset + i, stddev, seed, sid);
    }
}

unsigned grid_for(int64_t n, int threads) {
    int64_t g = (n + threads - 1) / threads;
    if (g > 148 * 32) g = 148 * 32;
    if (g < 1) g = 1;
    return static_cast<unsigned>(g);
}

__global__ void narrow_kernel(const int64_t* __restrict__ src, int32_t* __restrict__ dst, int64_t n) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        dst[i] = static_cast<int32_t>(src[i]);
}

// one warp per row; rows are k int32 (k % 4 == 0: 16-byte copies)
__global__ void scatter_rows_kernel(const int32_t* __restrict__ src, int32_t* __restrict__ dst,
                                    const int64_t* __restrict__ dst_row, int64_t nrows, int64_t row_elems) {
    const int lane = threadIdx.x & 31;
    const bool vec = (row_elems & 3) == 0;
    for (int64_t r = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5; r < nrows;
         r += (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5) {
        const int32_t* s = src + r * row_elems;
        int32_t* d = dst + __ldg(dst_row + r) * row_elems;
        if (vec) {
            for (int64_t i = lane; i < row_elems / 4; i += 32)
                reinterpret_cast<int4*>(d)[i] = __ldg(reinterpret_cast<const int4*>(s) + i);
        } else {
            for (int64_t i = lane; i < row_elems; i += 32) d[i] = __ldg(s + i);
        }
    }
}

}  // namespace

namespace csaidx_kern {

cudaError_t launch_narrow(const int64_t* src, int32_t* dst, int64_t n, cudaStream_t stream) {
    if (n <= 0) return cudaSuccess;
    narrow_kernel<<<grid_for(n, 256), 256, 0, stream>>>(src, dst, n);
    return cudaGetLastError();
}

cudaError_t launch_scatter_rows(const int32_t* src, int32_t* dst, const int64_t* dst_row, int64_t nrows,
                                int64_t row_elems, cudaStream_t stream) {
    if (nrows <= 0) return cudaSuccess;
    scatter_rows_kernel<<<grid_for(nrows * 32, 256), 256, 0, stream>>>(src, dst, dst_row, nrows, row_elems);
    return cudaGetLastError();
}


cudaError_t launch_convert_bf16(const ConvertParams& p, cudaStream_t stream) {
    if (p.n <= 0) return cudaSuccess;
    convert_bf16_kernel<<<grid_for(p.n, 256), 256, 0, stream>>>(p);
    return cudaGetLastError();
}

cudaError_t launch_fill_sentinel(float* val, int32_t* idx, int64_t n, cudaStream_t stream) {
    if (n <= 0) return cudaSuccess;
    fill_sentinel_kernel<<<grid_for(n, 256), 256, 0, stream>>>(val, idx, n);
    return cudaGetLastError();
}

cudaError_t launch_bool_mask(uint8_t* keep, int64_t rows, int64_t cols, int64_t s0, int64_t t0, int64_t ratio,
                             cudaStream_t stream) {
    const int64_t n = rows * cols;
    if (n <= 0) return cudaSuccess;
    bool_mask_kernel<<<grid_for(n, 256), 256, 0, stream>>>(keep, rows, cols, s0, t0, ratio);
    return cudaGetLastError();
}

cudaError_t launch_apply_bool_mask(float* scores, int64_t ld, const uint8_t* keep, int64_t batch, int64_t rows,
                                   int64_t cols, cudaStream_t stream) {
    const int64_t n = batch * rows * cols;
    if (n <= 0) return cudaSuccess;
    apply_bool_mask_kernel<<<grid_for(n, 256), 256, 0, stream>>>(scores, ld, keep, batch, rows, cols);
    return cudaGetLastError();
}

cudaError_t launch_gen_normal_bf16(__nv_bfloat16* dst, int64_t n, double stddev, uint64_t seed,
                                   uint64_t stream_id, int64_t offset, cudaStream_t stream) {
    if (n <= 0) return cudaSuccess;
    gen_bf16_kernel<<<grid_for(n, 256), 256, 0, stream>>>(dst, n, stddev, seed, stream_id, offset);
    return cudaGetLastError();
}

cudaError_t launch_gen_normal_f32(float* dst, int64_t n, double stddev, uint64_t seed, uint64_t stream_id,
                                  int64_t offset, cudaStream_t stream) {
    if (n <= 0) return cudaSuccess;
    gen_f32_kernel<<<grid_for(n, 256), 256, 0, stream>>>(dst, n, stddev, seed, stream_id, offset);
    return cudaGetLastError();
}

}  // namespace csaidx_kern
