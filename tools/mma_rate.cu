// Dev microbenchmark: clocks per tcgen05.mma (cta_group::1, kind::f16, bf16 -> fp32) for the
// shapes the attention kernel issues.  One CTA per SM, one thread issues `iters` MMAs
// back-to-back into one TMEM accumulator, commits, waits; reports clk per MMA and the
// implied FLOP/clk/SM.  Operands are uninitialised shared memory (timing only).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2511_06247_b200/csrc tools/mma_rate.cu -o /tmp/mma_rate
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#include "ptx.cuh"

using namespace cdsp::ptx;

template <int M, int N, bool TS, bool MN_B, int NACC>
__global__ void __launch_bounds__(128, 1) mma_rate(int iters, unsigned long long* out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint32_t slot;
    __shared__ __align__(8) uint64_t bar;
    const int warp = threadIdx.x / 32;
    if (warp == 0) {
        tmem_alloc(smem_u32(&slot), 512);
        tmem_relinquish();
    }
    if (threadIdx.x == 32) {
        mbar_init(smem_u32(&bar), 1);
        fence_barrier_init();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = slot;
    if (threadIdx.x == 0) {
        const uint32_t base = smem_u32(smem);
        const uint64_t da = umma_desc_sw128(base, 16, 1024);
        const uint64_t db = umma_desc_sw128(base + 65536, MN_B ? 16384 : 16, 1024);
        constexpr uint32_t idesc = idesc_bf16_f32(M, N, false, MN_B);
        const unsigned long long t0 = clock64();
        for (int i = 0; i < iters; ++i) {
            const uint64_t off = static_cast<uint64_t>((i & 3) * 2);
            const uint32_t acc = static_cast<uint32_t>((i % NACC) * N);  // NACC independent accumulators
            if (TS)
                mma_ts(tmem + 256 + (acc & 255), tmem + (i & 3) * 8, db + off, idesc, 1u);
            else
                mma_ss(tmem + acc, da + off, db + off, idesc, 1u);
        }
        mma_commit(smem_u32(&bar));
        mbar_wait(smem_u32(&bar), 0);
        const unsigned long long t1 = clock64();
        if (blockIdx.x == 0) out[0] = t1 - t0;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

template <int M, int N, bool TS, bool MN_B, int NACC = 1>
void run(const char* name, unsigned long long* d) {
    const int iters = 4096;
    auto k = mma_rate<M, N, TS, MN_B, NACC>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    k<<<148, 128, 160 * 1024>>>(iters, d);
    k<<<148, 128, 160 * 1024>>>(iters, d);
    unsigned long long h = 0;
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    const double clk = static_cast<double>(h) / iters;
    const double flop = 2.0 * M * N * 16;
    printf("%-34s %7.1f clk/MMA  %7.0f FLOP/clk/SM  (%s)\n", name, clk, flop / clk, cudaGetErrorString(cudaGetLastError()));
}

int main() {
    unsigned long long* d;
    cudaMalloc(&d, 8);
    run<128, 64, false, false>("SS M128 N64  (QK, BN=64)", d);
    run<128, 128, false, false>("SS M128 N128 (QK, BN=128)", d);
    run<128, 256, false, false>("SS M128 N256", d);
    run<128, 128, true, true>("TS M128 N128 B MN-major (PV)", d);
    run<128, 64, true, true>("TS M128 N64  B MN-major", d);
    run<128, 256, true, true>("TS M128 N256 B MN-major", d);
    run<128, 128, false, true>("SS M128 N128 B MN-major", d);
    run<128, 64, false, false, 2>("SS M128 N64  2 accumulators", d);
    run<128, 64, false, false, 4>("SS M128 N64  4 accumulators", d);
    run<128, 64, true, true, 2>("TS M128 N64  2 accumulators", d);
    run<128, 96, false, false>("SS M128 N96", d);
    run<128, 32, false, false, 4>("SS M128 N32  4 accumulators", d);
    run<128, 128, false, false, 2>("SS M128 N128 2 accumulators", d);
    return 0;
}
