// Dev microbenchmark: tensor-pipe time per 128x128 attention tile for the exact MMA pattern
// of attn_tc.cu (HD = 128): S = Q K^T as 8 SS MMAs (M=128, N=128, K=16, both K-major SW128)
// and O += P V as 8 TS MMAs (A = P from TMEM, B = V MN-major SW128), optionally with bulk
// copies streaming 64 KB per tile into shared memory (the K/V loads of the real kernel).
// One CTA per SM; thread 0 issues, thread 32 issues the bulk copies.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2511_06247_b200/csrc tools/mma_pattern.cu -o /tmp/mma_pattern
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#include "ptx.cuh"

using namespace cdsp::ptx;
__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

constexpr int kBox = 128 * 128;
constexpr int TILE = 2 * kBox;  // 128 rows x 128 bf16

__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(bar)
                 : "memory");
}

// mode bit 0: S MMAs, bit 1: PV MMAs, bit 2: concurrent bulk copies (64 KB / tile),
// bit 3: fill Q/K/V (and P) with random bf16 first (zeros otherwise),
// bit 4: warp-uniform loop as in attn_tc.cu (whole warp waits on an already-completed
//        mbarrier before each group, elect_one issues, __syncwarp after)
template <int MODE>
__global__ void __launch_bounds__(64, 1) pattern(int tiles, const uint8_t* gsrc, unsigned long long* out, int delay) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    __shared__ uint32_t slot;
    __shared__ __align__(8) uint64_t bars[4];
    const int warp = threadIdx.x / 32;
    if (warp == 0) {
        tmem_alloc(smem_u32(&slot), 512);
        tmem_relinquish();
    }
    if (threadIdx.x == 32) {
        for (int i = 0; i < 4; ++i) mbar_init(smem_u32(&bars[i]), 1);
        fence_barrier_init();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = slot;
    const uint32_t sQ = smem_u32(smem), sK = sQ + TILE, sV = sK + TILE, sL = sV + TILE;  // sL: copy target (64 KB)
    if (MODE & 8) {  // random bf16 in [-2, 2): data-dependent tensor-core power
        uint32_t* w = reinterpret_cast<uint32_t*>(smem);
        for (int i = threadIdx.x; i < 3 * TILE / 4; i += blockDim.x) {
            uint32_t x = (i + 1) * 2654435761u ^ (blockIdx.x * 40503u);
            x ^= x >> 13; x *= 0x5bd1e995u; x ^= x >> 15;
            const uint32_t lo = 0x3f80u | ((x & 0x7fu)) | ((x >> 7 & 1u) << 15) | ((x >> 8 & 1u) << 7);
            const uint32_t hi = 0x3f80u | ((x >> 16) & 0x7fu) | ((x >> 23 & 1u) << 15) | ((x >> 24 & 1u) << 7);
            w[i] = lo | (hi << 16);
        }
        __syncthreads();
        if (warp == 0) {  // P (bf16 pairs) in the three S buffers, O zero
            uint32_t v[16];
            for (int i = 0; i < 16; ++i) v[i] = 0x3f003f00u ^ ((threadIdx.x * 16 + i) * 0x00410041u & 0x007f007fu);
            for (int c = 128; c < 512; c += 16) tmem_st16(tmem + c, v);
            tc_wait_st();
        }
        tc_fence_before();
        __syncthreads();
        tc_fence_after();
    }
    if ((MODE & 16) && warp == 0 && (!(MODE & 32) || lane_id() == 0)) {
        constexpr uint32_t idesc_qk = idesc_bf16_f32(128, 128, false, false);
        constexpr uint32_t idesc_pv = idesc_bf16_f32(128, 128, false, true);
        const uint64_t dq = umma_desc_sw128(sQ, 16, 1024), dk = umma_desc_sw128(sK, 16, 1024);
        const uint64_t dv = umma_desc_sw128(sV, kBox, 1024);
        // bars[3]: complete phase 0 once so every later wait(parity 0) is already satisfied
        if ((((MODE & 32) != 0) || elect_one())) mbar_arrive(smem_u32(&bars[3]));
        if (!(MODE & 32)) __syncwarp();
        const unsigned long long t0 = clock64();
        for (int t = 0; t < tiles; ++t) {
            // bit 8: the CDSP_HALFSLOT placement (S in 64-column halves {0,1},{3,4},{1,2},{4,5}, P in 0/3/2/5)
            const int hs_h[4] = {0, 3, 1, 4}, hs_p[4] = {0, 3, 2, 5};
            const uint32_t sb = (MODE & 256) ? 128 + 64 * hs_h[t % 4] : 128 + 128 * (t % 3);
            const uint32_t sp = (MODE & 256) ? 128 + 64 * hs_p[t % 4] : sb;
            mbar_wait(smem_u32(&bars[3]), 0);
            mbar_wait(smem_u32(&bars[3]), 0);
            if (!(MODE & 64)) tc_fence_after();
            if ((((MODE & 32) != 0) || elect_one())) {
#pragma unroll
                for (int kk = 0; kk < 8; ++kk)
                    mma_ts(tmem, tmem + sp + kk * 8, dv + static_cast<uint64_t>((kk * 16 * 128) >> 4), idesc_pv, 1u);
                mma_commit(smem_u32(&bars[1]));
                if (!(MODE & 128)) mma_commit(smem_u32(&bars[1]));
            }
            if (!(MODE & 32)) __syncwarp();
            mbar_wait(smem_u32(&bars[3]), 0);
            if (!(MODE & 64)) tc_fence_after();
            if ((((MODE & 32) != 0) || elect_one())) {
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) {
                    const uint64_t off = static_cast<uint64_t>(((kk / 4) * kBox + (kk % 4) * 32) >> 4);
                    mma_ss(tmem + sb, dq + off, dk + off, idesc_qk, kk > 0 ? 1u : 0u);
                }
                mma_commit(smem_u32(&bars[0]));
                if (!(MODE & 128)) mma_commit(smem_u32(&bars[0]));
            }
            if (!(MODE & 32)) __syncwarp();
        }
        if ((((MODE & 32) != 0) || elect_one())) mma_commit(smem_u32(&bars[2]));
        if (!(MODE & 32)) __syncwarp();
        mbar_wait(smem_u32(&bars[2]), 0);
        const unsigned long long t1 = clock64();
        if (blockIdx.x == 0 && lane_id() == 0) out[0] = t1 - t0;
    } else if (!(MODE & 16) && threadIdx.x == 0) {
        constexpr uint32_t idesc_qk = idesc_bf16_f32(128, 128, false, false);
        constexpr uint32_t idesc_pv = idesc_bf16_f32(128, 128, false, true);
        const uint64_t dq = umma_desc_sw128(sQ, 16, 1024), dk = umma_desc_sw128(sK, 16, 1024);
        const uint64_t dv = umma_desc_sw128(sV, kBox, 1024);
        const unsigned long long t0 = clock64();
        for (int t = 0; t < tiles; ++t) {
            // bit 8: the CDSP_HALFSLOT placement (S in 64-column halves {0,1},{3,4},{1,2},{4,5}, P in 0/3/2/5)
            const int hs_h[4] = {0, 3, 1, 4}, hs_p[4] = {0, 3, 2, 5};
            const uint32_t sb = (MODE & 256) ? 128 + 64 * hs_h[t % 4] : 128 + 128 * (t % 3);
            const uint32_t sp = (MODE & 256) ? 128 + 64 * hs_p[t % 4] : sb;
            if (MODE & 1) {
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) {
                    const uint64_t off = static_cast<uint64_t>(((kk / 4) * kBox + (kk % 4) * 32) >> 4);
                    mma_ss(tmem + sb, dq + off, dk + off, idesc_qk, kk > 0 ? 1u : 0u);
                }
                mma_commit(smem_u32(&bars[0]));
                if (delay) {  // issuer busy for `delay` clk after the group (a barrier wait, ...)
                    const unsigned long long d0 = clock64();
                    while (clock64() - d0 < static_cast<unsigned long long>(delay)) {
                    }
                }
            }
            if (MODE & 2) {
#pragma unroll
                for (int kk = 0; kk < 8; ++kk)
                    mma_ts(tmem, tmem + sp + kk * 8, dv + static_cast<uint64_t>((kk * 16 * 128) >> 4), idesc_pv, 1u);
                mma_commit(smem_u32(&bars[1]));
                if (delay) {
                    const unsigned long long d0 = clock64();
                    while (clock64() - d0 < static_cast<unsigned long long>(delay)) {
                    }
                }
            }
        }
        mma_commit(smem_u32(&bars[2]));
        mbar_wait(smem_u32(&bars[2]), 0);
        const unsigned long long t1 = clock64();
        if (blockIdx.x == 0) out[0] = t1 - t0;
    } else if ((MODE & 4) && threadIdx.x == 32) {
        // stream 64 KB per "tile" into sL, as fast as the copy engine allows, until told to stop
        const uint8_t* src = gsrc + static_cast<size_t>(blockIdx.x % 16) * 65536;
        for (int t = 0; t < tiles; ++t) {
            mbar_expect_tx(smem_u32(&bars[3]), 65536);
            bulk_g2s(sL, src, 65536, smem_u32(&bars[3]));
            mbar_wait(smem_u32(&bars[3]), t & 1);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

template <int MODE>
void run(const char* name, const uint8_t* g, unsigned long long* d, int delay = 0) {
    const int tiles = 2000;
    auto k = pattern<MODE>;
    const int smem = 3 * TILE + 65536 + 1024;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    k<<<148, 64, smem>>>(tiles, g, d, delay);
    k<<<148, 64, smem>>>(tiles, g, d, delay);
    unsigned long long h = 0;
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    const double clk = static_cast<double>(h) / tiles;
    const int nmma = (MODE & 16) ? 16 : ((MODE & 1) ? 8 : 0) + ((MODE & 2) ? 8 : 0);
    printf("%-44s %7.1f clk/tile  %6.1f clk/MMA  (%s)\n", name, clk, clk / nmma, cudaGetErrorString(cudaGetLastError()));
}

int main() {
    unsigned long long* d;
    uint8_t* g;
    cudaMalloc(&d, 8);
    cudaMalloc(&g, 16 * 65536);
    cudaMemset(g, 0, 16 * 65536);
    run<1>("S only (8 SS, N=128)", g, d);
    run<2>("PV only (8 TS, V MN-major, N=128)", g, d);
    run<3>("S + PV (ideal 1024)", g, d);
    run<5>("S only + 64 KB/tile bulk copies", g, d);
    run<6>("PV only + 64 KB/tile bulk copies", g, d);
    run<7>("S + PV + 64 KB/tile bulk copies", g, d);
    run<9>("S only, random data", g, d);
    run<10>("PV only, random data", g, d);
    run<11>("S + PV, random data", g, d);
    run<15>("S + PV + copies, random data", g, d);
    run<16>("warp loop: 3 waits + elect + 4 commits / tile", g, d);
    run<16 + 32>("lane-0 loop: 3 waits + 4 commits / tile", g, d);
    run<16 + 64>("warp loop, no tcgen05 fence", g, d);
    run<16 + 128>("warp loop, 2 commits / tile", g, d);
    run<16 + 32 + 64 + 128>("lane-0, no fence, 2 commits", g, d);
    run<3 + 256>("S + PV, half-slot placement", g, d);
    run<11 + 256>("S + PV, half-slot placement, random data", g, d);
    run<3>("S + PV, issuer +50 clk per group", g, d, 50);
    run<3>("S + PV, issuer +100 clk per group", g, d, 100);
    run<3>("S + PV, issuer +200 clk per group", g, d, 200);
    run<3>("S + PV, issuer +400 clk per group", g, d, 400);
    run<3>("S + PV, issuer +500 clk per group", g, d, 500);
    return 0;
}
