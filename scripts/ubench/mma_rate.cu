// (dev) tcgen05.mma issue-to-completion throughput vs N, SS and TS (A from
// TMEM) forms, M = 128, K = 16 per instruction, bf16 -> fp32. One CTA per SM,
// one thread issues `iters` MMAs into one accumulator, commit, wait; cycles
// per MMA printed. Operand contents are irrelevant (zeros).
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include "../../paper_2605_02568_b200/csrc/kernels/sm100_ptx.cuh"
using namespace csaidx_dev;

__device__ __forceinline__ void umma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}"
                 :: "r"(d), "r"(a), "l"(b), "r"(idesc), "r"(acc));
}

template <int N, bool TS>
__global__ void __launch_bounds__(128, 1) k_mma(long long* out, int iters) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    __shared__ uint64_t bar;
    __shared__ uint32_t tslot;
    for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
    if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
    if (threadIdx.x < 32) tmem_alloc<512>(&tslot);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tslot;
    if (threadIdx.x == 0) {
        const uint32_t a = smem_u32(smem), bb = smem_u32(smem + 32 * 1024);
        constexpr uint32_t idesc = idesc_bf16_f32(128, N);
        long long t0 = clock64();
        for (int i = 0; i < iters; ++i) {
            const uint32_t kk = i & 3;
            if (TS) umma_ts(tmem + 256, tmem + 0 + kk * 8, sw128_kmajor_desc(bb + kk * 32), idesc, i > 0);
            else umma_bf16(tmem + 256, sw128_kmajor_desc(a + kk * 32), sw128_kmajor_desc(bb + kk * 32), idesc, i > 0);
        }
        umma_commit(&bar);
        mbar_wait(&bar, 0);
        long long t1 = clock64();
        out[blockIdx.x] = t1 - t0;
    }
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x < 32) { tc_fence_after(); tmem_dealloc<512>(tmem); }
}

template <int N, bool TS>
void run(long long* d, int iters, int grid) {
    cudaFuncSetAttribute(k_mma<N, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65 * 1024);
    k_mma<N, TS><<<grid, 128, 65 * 1024>>>(d, iters);
    k_mma<N, TS><<<grid, 128, 65 * 1024>>>(d, iters);
    cudaDeviceSynchronize();
    long long h[148];
    cudaMemcpy(h, d, grid * sizeof(long long), cudaMemcpyDeviceToHost);
    double s = 0; for (int i = 0; i < grid; ++i) s += h[i];
    printf("N=%3d %s: %.1f cycles per MMA (%.0f MAC/cycle/SM)  err=%s\n", N, TS ? "TS (A in TMEM)" : "SS          ",
           s / grid / iters, 128.0 * N * 16 / (s / grid / iters), cudaGetErrorString(cudaGetLastError()));
}

int main() {
    long long* d; cudaMalloc(&d, 148 * sizeof(long long));
    const int it = 4096, grid = 148;
    run<16, false>(d, it, grid); run<32, false>(d, it, grid); run<64, false>(d, it, grid);
    run<128, false>(d, it, grid); run<256, false>(d, it, grid);
    run<16, true>(d, it, grid); run<32, true>(d, it, grid); run<64, true>(d, it, grid);
    run<128, true>(d, it, grid); run<256, true>(d, it, grid);
    return 0;
}
