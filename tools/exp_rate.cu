// Dev microbenchmark (both operands loop-variant so nothing is hoisted; measured on B200:
// MUFU.EX2 issues at 16 lanes/clk/SM, so exp2 of a 128x128 tile costs 1024 SM clocks --
// the same as the tile's two M=128,N=128,K=128 MMAs).  Throughput of the softmax exponential block (32 scores -> 16 packed
// bf16 pairs, FFMA2 + MUFU.EX2 / FMA-pipe cubic + FADD2 + F2FP) with 16 warps per SM
// (4 per SMSP), registers only.  Reports SM clocks per block per warp-quad (= one 128-key
// tile of the attention kernel's softmax on one SMSP).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2511_06247_b200/csrc -I include tools/exp_rate.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#include "ptx.cuh"

using namespace cdsp::ptx;

__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
    float2 d;
    asm("{\n\t.reg .b64 ra, rb, rc, rd;\n\tmov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\tmov.b64 rc, {%6, %7};\n\t"
        "fma.rn.f32x2 rd, ra, rb, rc;\n\tmov.b64 {%0, %1}, rd;\n\t}"
        : "=f"(d.x), "=f"(d.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
    return d;
}
__device__ __forceinline__ float2 fadd2(float2 a, float2 b) {
    float2 d;
    asm("{\n\t.reg .b64 ra, rb, rd;\n\tmov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
        "add.f32x2 rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;\n\t}"
        : "=f"(d.x), "=f"(d.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
    return d;
}
__device__ __forceinline__ float2 ex2_fma2(float2 x) {
    x.x = fmaxf(x.x, -126.0f);
    x.y = fmaxf(x.y, -126.0f);
    const float2 t = fadd2(x, make_float2(12582912.0f, 12582912.0f));
    const float2 n = fadd2(t, make_float2(-12582912.0f, -12582912.0f));
    const float2 f = fadd2(x, make_float2(-n.x, -n.y));
    float2 q = ffma2(make_float2(0.0551713891f, 0.0551713891f), f, make_float2(0.2426107079f, 0.2426107079f));
    q = ffma2(q, f, make_float2(0.6932609677f, 0.6932609677f));
    q = ffma2(q, f, make_float2(0.9999281168f, 0.9999281168f));
    return make_float2(__int_as_float(__float_as_int(q.x) + (__float_as_int(t.x) << 23)),
                       __int_as_float(__float_as_int(q.y) + (__float_as_int(t.y) << 23)));
}

template <int MASK, bool PACKED>
__global__ void __launch_bounds__(512, 1) exp_rate(int iters, const float* in, uint32_t* out, unsigned long long* clk) {
    uint32_t s[32];
    for (int i = 0; i < 32; ++i) s[i] = __float_as_uint(in[(threadIdx.x + i) & 255]);
    float2 lacc = make_float2(0.f, 0.f);
    uint32_t acc = 0;
    const float sl2 = 0.127f, m_use = 3.0f;
    __syncthreads();
    const unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        const float2 sc = make_float2(sl2, sl2), nm = make_float2(-m_use - it * 1e-7f, -m_use - it * 2e-7f);  // both lanes loop-variant (no hoisting)
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            float2 x;
            if (PACKED) {
                x = ffma2(make_float2(__uint_as_float(s[2 * i]), __uint_as_float(s[2 * i + 1])), sc, nm);
            } else {
                x = make_float2(fmaf(__uint_as_float(s[2 * i]), sl2, nm.x), fmaf(__uint_as_float(s[2 * i + 1]), sl2, nm.y));
            }
            float2 pp;
            if ((MASK >> (i % 8)) & 1) {
                pp = ex2_fma2(x);
            } else {
                pp.x = ex2(x.x);
                pp.y = ex2(x.y);
            }
            if (PACKED) lacc = fadd2(lacc, pp);
            else { lacc.x += pp.x; lacc.y += pp.y; }
            acc ^= pack_bf16(pp.x, pp.y);
        }
    }
    const unsigned long long t1 = clock64();
    out[blockIdx.x * 512 + threadIdx.x] = acc ^ __float_as_uint(lacc.x + lacc.y);
    if (threadIdx.x == 0 && blockIdx.x == 0) *clk = t1 - t0;
}

template <int MASK, bool PACKED>
void run(const char* name, const float* in, uint32_t* out, unsigned long long* d, int wps = 4) {
    const int iters = 2000;  // wps: warps per SMSP (1: one warp's latency-bound stream, as a softmax group's)
    exp_rate<MASK, PACKED><<<148, 128 * wps>>>(iters, in, out, d);
    exp_rate<MASK, PACKED><<<148, 128 * wps>>>(iters, in, out, d);
    unsigned long long h;
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("%-40s %7.1f clk per 32-score block per SMSP (%d warp%s)  [%s]\n", name, double(h) / iters, wps,
           wps > 1 ? "s" : "", cudaGetErrorString(cudaGetLastError()));
}

int main() {
    float* in;
    uint32_t* out;
    unsigned long long* d;
    cudaMalloc(&in, 256 * 4);
    cudaMalloc(&out, 148 * 512 * 4);
    cudaMalloc(&d, 8);
    cudaMemset(in, 0, 256 * 4);
    run<0x00, true>("all MUFU, packed", in, out, d);
    run<0x22, true>("1/4 FMA cubic, packed", in, out, d);
    run<0x52, true>("3/8 FMA cubic, packed", in, out, d);
    run<0x55, true>("1/2 FMA cubic, packed", in, out, d);
    run<0xFF, true>("all FMA cubic, packed", in, out, d);
    run<0x00, false>("all MUFU, scalar FFMA/FADD", in, out, d);
    run<0x52, false>("3/8 FMA cubic, scalar", in, out, d);
    for (int w = 1; w <= 4; w *= 2) {  // latency vs throughput of the kernel's 1/8 mix
        run<0x02, true>("1/8 FMA cubic, packed", in, out, d, w);
        run<0x00, true>("all MUFU, packed", in, out, d, w);
        run<0x22, true>("1/4 FMA cubic, packed", in, out, d, w);
    }
    return 0;
}
