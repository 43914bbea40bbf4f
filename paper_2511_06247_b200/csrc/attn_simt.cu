// attn_simt.cu — K*2: fp32 block attention on the FFMA pipes (the fp32 path of the
// north_star: 1e-4 max-abs; single-pass TF32 tensor cores miss that bound, R12).
//
// Same contract as the tcgen05 kernel (segments, modes, LSE merge epilogue).  One thread
// owns one query row: its O row lives in registers, Q is staged transposed in shared
// memory (conflict-free), K/V tiles are broadcast from shared memory.
#include <cuda_runtime.h>

#include "attn_common.cuh"
#include "common.cuh"
#include "internal.h"

namespace cdsp {
namespace {

constexpr int SB_M = 64;  // query rows per block (one per thread)
constexpr int SB_N = 16;  // KV rows per tile (48 KB static smem at HD=128)

struct SimtParams {
    const float* q;
    const float* k;
    const float* v;
    cdsp_segments seg;
    int Hq, Hkv, g, n_rb;
    float scale_log2;
    int mode;
    float* o_acc;
    float* lse_acc;
    float* out;
    float* lse;
};

template <int HD>
__global__ void __launch_bounds__(SB_M) attn_simt_kernel(const SimtParams p) {
    __shared__ float sQt[HD][SB_M];
    __shared__ __align__(16) float sK[SB_N][HD];
    __shared__ __align__(16) float sV[SB_N][HD];
    const cdsp_segments& sg = p.seg;
    const int rb = p.n_rb - 1 - blockIdx.x / p.Hq;
    const int h = blockIdx.x % p.Hq;
    const int kvh = h / p.g;
    const int tid = threadIdx.x;
    const int64_t row0 = static_cast<int64_t>(rb) * SB_M;
    const int64_t row = row0 + tid;
    const bool row_ok = row < sg.nq;
    const int64_t my_qpos = row_ok ? seg_qpos(sg, row) : INT64_MAX;
    int64_t qlo, qhi;
    bool qany;
    seg_qrange(sg, row0, row0 + SB_M, qlo, qhi, qany);

    // stage Q^T
    for (int idx = tid; idx < SB_M * HD; idx += SB_M) {
        const int r = idx / HD, d = idx % HD;
        const int64_t gr = row0 + r;
        sQt[d][r] = gr < sg.nq ? p.q[(static_cast<size_t>(gr) * p.Hq + h) * HD + d] : 0.f;
    }
    float o[HD];
#pragma unroll
    for (int d = 0; d < HD; ++d) o[d] = 0.f;
    float m = -INFINITY, l = 0.f;
    const float sl2 = p.scale_log2;
    const int n_tiles = static_cast<int>((sg.nkv + SB_N - 1) / SB_N);
    for (int j = 0; j < n_tiles; ++j) {
        const int64_t c0 = static_cast<int64_t>(j) * SB_N;
        const int kind = seg_tile_kind(sg, qany, qlo, qhi, c0, SB_N);
        if (kind == TILE_EMPTY) continue;  // block-uniform
        __syncthreads();
        for (int idx = tid; idx < SB_N * HD / 4; idx += SB_M) {
            const int r = idx / (HD / 4), d4 = idx % (HD / 4);
            const int64_t gr = c0 + r;
            float4 kk = make_float4(0.f, 0.f, 0.f, 0.f), vv = kk;
            if (gr < sg.nkv) {
                kk = reinterpret_cast<const float4*>(p.k + (static_cast<size_t>(gr) * p.Hkv + kvh) * HD)[d4];
                vv = reinterpret_cast<const float4*>(p.v + (static_cast<size_t>(gr) * p.Hkv + kvh) * HD)[d4];
            }
            reinterpret_cast<float4*>(&sK[r][0])[d4] = kk;
            reinterpret_cast<float4*>(&sV[r][0])[d4] = vv;
        }
        __syncthreads();
        float s[SB_N];
#pragma unroll
        for (int c = 0; c < SB_N; ++c) s[c] = 0.f;
#pragma unroll 4
        for (int d = 0; d < HD; d += 4) {
            const float q0 = sQt[d][tid], q1 = sQt[d + 1][tid], q2 = sQt[d + 2][tid], q3 = sQt[d + 3][tid];
#pragma unroll
            for (int c = 0; c < SB_N; ++c) {
                const float4 kk = *reinterpret_cast<const float4*>(&sK[c][d]);
                s[c] = fmaf(q0, kk.x, fmaf(q1, kk.y, fmaf(q2, kk.z, fmaf(q3, kk.w, s[c]))));
            }
        }
        float mx = -INFINITY;
#pragma unroll
        for (int c = 0; c < SB_N; ++c) {
            if (kind == TILE_PARTIAL && !seg_visible(sg, c0 + c, my_qpos)) s[c] = -INFINITY;
            mx = fmaxf(mx, s[c]);
        }
        const float m_new = fmaxf(m, mx * sl2);
        const float m_use = (m_new == -INFINITY) ? 0.f : m_new;
        const float alpha = exp2f(m - m_use);  // m = -inf -> 0
        l *= alpha;
#pragma unroll
        for (int d = 0; d < HD; ++d) o[d] *= alpha;
        m = m_new;
#pragma unroll
        for (int c = 0; c < SB_N; ++c) {
            const float pc = exp2f(fmaf(s[c], sl2, -m_use));
            l += pc;
#pragma unroll
            for (int d = 0; d < HD; d += 4) {
                const float4 vv = *reinterpret_cast<const float4*>(&sV[c][d]);
                o[d] = fmaf(pc, vv.x, o[d]);
                o[d + 1] = fmaf(pc, vv.y, o[d + 1]);
                o[d + 2] = fmaf(pc, vv.z, o[d + 2]);
                o[d + 3] = fmaf(pc, vv.w, o[d + 3]);
            }
        }
    }
    if (!row_ok) return;
    const float inv_l = l > 0.f ? 1.0f / l : 0.f;
    const float lse_b = l > 0.f ? (m + log2f(l)) * 0.69314718055994530942f : -INFINITY;
    const size_t orow = (static_cast<size_t>(row) * p.Hq + h) * HD;
    const size_t li = static_cast<size_t>(h) * sg.nq + row;
    float wa = 0.f, wb = 1.f, lse_out = lse_b;
    if (p.mode == CDSP_ATTN_MID || p.mode == CDSP_ATTN_LAST) {
        // accurate expf/logf on the fp32 path
        const float lse_a = p.lse_acc[li];
        const float M = fmaxf(lse_a, lse_b);
        if (M == -INFINITY) {
            wa = wb = 0.f;
            lse_out = -INFINITY;
        } else {
            const float ea = expf(lse_a - M), eb = expf(lse_b - M);
            wa = ea / (ea + eb);
            wb = eb / (ea + eb);
            lse_out = M + logf(ea + eb);
        }
    }
    const float sb = wb * inv_l;
    float* dst = (p.mode == CDSP_ATTN_FIRST || p.mode == CDSP_ATTN_MID) ? p.o_acc : p.out;
#pragma unroll
    for (int d = 0; d < HD; d += 4) {
        float4 r4 = make_float4(o[d] * sb, o[d + 1] * sb, o[d + 2] * sb, o[d + 3] * sb);
        if (p.mode == CDSP_ATTN_MID || p.mode == CDSP_ATTN_LAST) {
            const float4 a = *reinterpret_cast<const float4*>(p.o_acc + orow + d);
            r4.x = fmaf(wa, a.x, r4.x);
            r4.y = fmaf(wa, a.y, r4.y);
            r4.z = fmaf(wa, a.z, r4.z);
            r4.w = fmaf(wa, a.w, r4.w);
        }
        *reinterpret_cast<float4*>(dst + orow + d) = r4;
    }
    if (p.mode == CDSP_ATTN_FIRST || p.mode == CDSP_ATTN_MID)
        p.lse_acc[li] = lse_out;
    else if (p.lse)
        p.lse[li] = lse_out;
}

template <int HD>
cdsp_status launch_simt(const AttnArgs& a, cudaStream_t st) {
    SimtParams p;
    p.q = static_cast<const float*>(a.q);
    CDSP_REQUIRE(a.nblk == 1, CDSP_ERR_UNSUPPORTED, "the fp32 kernel takes one KV block per launch");
    p.k = static_cast<const float*>(a.k[0]);
    p.v = static_cast<const float*>(a.v[0]);
    p.seg = a.seg[0];
    p.Hq = a.Hq;
    p.Hkv = a.Hkv;
    p.g = a.Hq / a.Hkv;
    p.n_rb = static_cast<int>((a.seg[0].nq + SB_M - 1) / SB_M);
    p.scale_log2 = a.scale * 1.4426950408889634f;
    p.mode = a.mode;
    p.o_acc = a.o_acc;
    p.lse_acc = a.lse_acc;
    p.out = static_cast<float*>(a.out);
    p.lse = a.lse;
    const int64_t grid = static_cast<int64_t>(p.n_rb) * a.Hq;
    if (grid == 0) return CDSP_OK;
    CDSP_REQUIRE(grid < (1ll << 31), CDSP_ERR_SHAPE, "grid too large");
    attn_simt_kernel<HD><<<static_cast<unsigned>(grid), SB_M, 0, st>>>(p);
    CDSP_CUDA(cudaGetLastError());
    return CDSP_OK;
}

}  // namespace

cdsp_status launch_attention_simt(const AttnArgs& a, cudaStream_t st) {
    if (a.D == 128) return launch_simt<128>(a, st);
    if (a.D == 64) return launch_simt<64>(a, st);
    CDSP_FAIL(CDSP_ERR_SHAPE, "head dim %d not supported (64 or 128)", a.D);
}

}  // namespace cdsp
