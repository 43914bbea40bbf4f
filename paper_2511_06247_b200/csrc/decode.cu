// decode.cu — the decode consumer of the transferred cache: one decode
// step's attention on one decode TP rank, read straight from the paged K/V cache that
// cdsp_kv_transfer_to_decode wrote (R15), as split-KV flash-decoding.
//
// The paper's decode instances run PagedAttention-style decoding over block-granular caches
// (§2.2 "PagedAttention ... block granularity"; §6 Tetris "reuses some
// components of vLLM") after the prefill streams each chunk's KV to them.
// A decode step's query (the newest token, position n_ctx - 1, whose K/V the decode
// instance has already appended) attends to every cached token: exact softmax attention,
// the same definition as the prefill (R1, R2, R14).
//
// B200 design.  One query row per head makes this a pure HBM stream: per token 2 Hkv_t D
// elements are read once and every byte feeds G = Hq_t/Hkv_t dot products, ~4 FLOP/B, far
// below any tensor-core ridge, so it is sized for bandwidth.  The bf16 paths compute S and PV
// with the legacy warp MMA (mma.sync m16n8k16: one query row per head leaves no M for a
// tcgen05 tile) and are fed by TMA page boxes (decode_tma_kernel, block size >= 16) or per-warp
// cp.async rings (decode_mma_kernel, any block size); the f32 path (decode_attn_kernel,
// described here) runs on the FMA pipe:
//  * grid = (n_split, Hkv_t), 256 threads; n_split x Hkv_t = one wave of resident CTAs
//    (occupancy x 148) so that every SM streams; each CTA owns a contiguous token range, its
//    8 warps interleave 8-vector steps.
//  * a warp step covers 8 x TPI tokens: lane (tsub, c) loads 16-byte vector c of token
//    i*TPI + tsub for i < 8 (for bf16 D=128: 16 lanes per 256-byte row, 2 rows per
//    instruction), K and V of the whole step issued before any use (16 x 16 B per lane in
//    flight, 64 KB per CTA), non-allocating in L1; block-table lookups per token (any power
//    of two block size, pages need not align with steps).
//  * q . k: per head, the lane's 8 partial dot products are reduce-scattered over the CPR
//    lanes of a row (7 shuffles instead of 32 for a plain butterfly), then the 8 full scores
//    are gathered back (8 shuffles), so every lane runs the online softmax of its token
//    slot locally (no cross-lane max) and P V needs no further exchange.
//  * partials: the CTA merges its 8 x TPI lane-group states in shared memory; splits merge
//    inside the same launch (merge_slice: the last finishers, column slices in parallel):
//    no second kernel, no host round trip.  Weights 2^(m_j - M) (R3 in base 2).
//  * a batch of requests (cdsp_decode_attention_batch, TMA kernel only): virtual heads =
//    (request, KV head) carry the merge state exactly as one request's KV heads do; the grid is
//    1D over every request's splits back to back (DecTmaBatchArgs: request offsets and lengths in
//    kernel-parameter space, found by binary search), sized to one wave over the whole batch.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstring>
#include <algorithm>

#include "common.cuh"
#include "internal.h"
#include "ptx.cuh"

namespace cdsp {
namespace {

#ifdef CDSP_DTRACE
// debug timeline (build with -DCDSP_DTRACE): per CTA globaltimer at start, after its own
// stream loop, after its CTA merge, at exit; read with cdsp_debug_decode_trace
__device__ unsigned long long g_dtrace[4096 * 8];
__device__ __forceinline__ void dstamp(int slot) {
    if (threadIdx.x == 0 && blockIdx.y == 0 && blockIdx.x < 4096) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        g_dtrace[blockIdx.x * 8 + slot] = t;
        if (slot == 0) {
            unsigned smid;
            asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
            g_dtrace[blockIdx.x * 8 + 7] = smid + 1;
        }
    }
}
#else
__device__ __forceinline__ void dstamp(int) {}
#endif

constexpr int kThreads = 256, kWarps = 8;
constexpr int kNI = 8;          // 16-byte vectors per lane per step (log2 = 3)
#ifndef CDSP_DEC_MERGE  // 1: slice-parallel merge by the last finishers; 0: two-level group merge
#define CDSP_DEC_MERGE 1
#endif
constexpr int kGroup = 16;      // splits merged by a level-1 merger (CDSP_DEC_MERGE = 0)
constexpr int kMaxSplit = 512;  // splits per KV head
constexpr int kMaxGroups = kMaxSplit / kGroup;

struct DecodeParams {
    const void* q;   // [Hq_t, D] ([batch, Hq_t, D] for a batch)
    const void* kc;  // [num_blocks, B, Hkv_t, D]
    const void* vc;
    const int32_t* bt;
    int64_t bt_stride;  // batch (TMA kernel): request b reads block-table row b, bt_stride entries apart
    int64_t num_blocks, n_ctx, tok_per_split;
    int b_shift, Hkv_t, n_split, n_groups;
    float scale_log2;
    float* o1;   // [Hkv_t][kMaxSplit][G][D]
    float* l1;   // [Hkv_t][kMaxSplit][G]   (log2-domain lse)
    float* o2;   // [Hkv_t][kMaxGroups][G][D]
    float* l2;   // [Hkv_t][kMaxGroups][G]
    int* cnt1;   // [Hkv_t][kMaxGroups]
    int* cnt2;   // [Hkv_t]
    void* out;   // [Hq_t, D]
    float* lse;  // [Hq_t] natural log, or NULL
};

__device__ __forceinline__ uint4 ld_stream(const void* p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}

template <typename T>
struct Vec;
template <>
struct Vec<__nv_bfloat16> {
    static constexpr int N = 8;
    __device__ static __forceinline__ void unpack(const uint4& u, float* f) {
        const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            f[2 * i] = __uint_as_float(w[i] << 16);
            f[2 * i + 1] = __uint_as_float(w[i] & 0xFFFF0000u);
        }
    }
    __device__ static __forceinline__ void store(__nv_bfloat16* p, float x) { *p = __float2bfloat16_rn(x); }
};
template <>
struct Vec<float> {
    static constexpr int N = 4;
    __device__ static __forceinline__ void unpack(const uint4& u, float* f) {
        f[0] = __uint_as_float(u.x);
        f[1] = __uint_as_float(u.y);
        f[2] = __uint_as_float(u.z);
        f[3] = __uint_as_float(u.w);
    }
    __device__ static __forceinline__ void store(float* p, float x) { *p = x; }
};

__device__ __forceinline__ float ex2f(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

__host__ __device__ constexpr int ilog2(int x) { return x <= 1 ? 0 : 1 + ilog2(x / 2); }

// Merge n <= 32 partial states (o normalised, lse in log2 units, -inf = empty) per (head, d):
// w_j = 2^(l_j - M) / sum_k 2^(l_k - M).  Whole CTA.  The partials were written by other CTAs
// moments ago, so every load bypasses L1 (ld.cg).  Latency, not bandwidth, decides this tail:
// every thread first issues ALL its o loads (16-byte vectors, one per partial), then the lse
// values are staged and the weights computed while those loads are in flight — one L2 round
// trip per merge instead of one per partial.
template <typename T, int HD, int G>
__device__ void merge_parts(const float* o_src, const float* l_src, int n, float* o_dst, float* l_dst, T* out,
                            float* lse, float* w_sh /* [32 * G] */, float* lse_sh /* [G] */) {
    constexpr int U = G * HD / 4;  // float4 units per partial
    const int tid = threadIdx.x;
    const int nthr = blockDim.x;
    constexpr int kMaxU = (U + 127) / 128;  // units per thread (blockDim >= 128)
    auto load = [&](int u, float4* v) {
#pragma unroll
        for (int j = 0; j < 32; ++j)
            v[j] = (j < n && u < U) ? __ldcg(reinterpret_cast<const float4*>(o_src + static_cast<size_t>(j) * G * HD) + u)
                                    : make_float4(0.f, 0.f, 0.f, 0.f);
    };
    auto weights = [&]() {
        for (int i = tid; i < n * G; i += nthr) w_sh[i] = __ldcg(l_src + i);
        __syncthreads();
        if (tid < G) {
            float M = -INFINITY;
            for (int j = 0; j < n; ++j) M = fmaxf(M, w_sh[j * G + tid]);
            float den = 0.f;
            for (int j = 0; j < n; ++j) {
                const float lj = w_sh[j * G + tid];
                const float w = lj == -INFINITY ? 0.f : ex2f(lj - M);
                w_sh[j * G + tid] = w;
                den += w;
            }
            const float inv = den > 0.f ? 1.f / den : 0.f;
            for (int j = 0; j < n; ++j) w_sh[j * G + tid] *= inv;
            lse_sh[tid] = den > 0.f ? M + __log2f(den) : -INFINITY;
        }
        __syncthreads();
    };
    auto combine = [&](int u, const float4* v) {
        if (u >= U) return;
        const int h = (4 * u) / HD;
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int j = 0; j < 32; ++j) {
            if (j < n) {  // empty partials hold o = 0 and weight 0
                const float w = w_sh[j * G + h];
                acc.x = fmaf(w, v[j].x, acc.x);
                acc.y = fmaf(w, v[j].y, acc.y);
                acc.z = fmaf(w, v[j].z, acc.z);
                acc.w = fmaf(w, v[j].w, acc.w);
            }
        }
        if (out) {
            Vec<T>::store(out + 4 * u, acc.x);
            Vec<T>::store(out + 4 * u + 1, acc.y);
            Vec<T>::store(out + 4 * u + 2, acc.z);
            Vec<T>::store(out + 4 * u + 3, acc.w);
        } else {
            reinterpret_cast<float4*>(o_dst)[u] = acc;
        }
    };
    float4 v[32];
    if constexpr (kMaxU == 1) {
        load(tid, v);  // in flight while the weights are computed
        weights();
        combine(tid, v);
    } else {
        weights();
        for (int k = 0; k < kMaxU; ++k) {
            load(tid + k * nthr, v);
            combine(tid + k * nthr, v);
        }
    }
    if (tid < G) {
        if (out) {
            if (lse) lse[tid] = lse_sh[tid] * 0.69314718055994530942f;
        } else {
            l_dst[tid] = lse_sh[tid];
        }
    }
}

// Split merge by the last finishers (CDSP_DEC_MERGE = 1).  Every split CTA has written its
// partial (o normalised, lse in log2 units); the partials are merged column-slice-parallel:
// slice sl = 8 consecutive elements of the [G][HD] output, merged over ALL n splits by one CTA
// (w_j = 2^(lse_j - M) / sum_k 2^(lse_k - M), R3 in base 2).  The CTAs doing it are the LAST K
// = min(G HD / 8, n) to finish (their finishing rank is an atomic count): each waits for the
// count to reach n (the others are resident: the grid is one wave) and merges slices q, q + K,
// ...  One L2 round trip for all of a slice's loads (n <= 512 partials: <= 4 lse and <= 8
// float4 per thread), instead of a two-level chain of merges after the last split.
template <typename T, int HD, int G>
__device__ void merge_slice(const DecodeParams& p, int kvh, int sl) {
    __shared__ float w_all[kMaxSplit];
    __shared__ float red[32];
    __shared__ float4 red4[32][2];
    const int tid = threadIdx.x, nt = blockDim.x, n = p.n_split;
    const int lane = tid & 31, wid = tid >> 5, nw = nt >> 5;
    const int c0 = sl * 8, h = c0 / HD, half = tid & 1, hn = nt >> 1;
    const float* l1 = p.l1 + static_cast<size_t>(kvh) * kMaxSplit * G + h;
    const float* o1 = p.o1 + static_cast<size_t>(kvh) * kMaxSplit * G * HD + c0 + 4 * half;
    float lv[4];
    float4 ov[8];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int j = tid + i * nt;
        lv[i] = j < n ? __ldcg(l1 + static_cast<size_t>(j) * G) : -INFINITY;
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int j = (tid >> 1) + i * hn;
        ov[i] = j < n ? __ldcg(reinterpret_cast<const float4*>(o1 + static_cast<size_t>(j) * G * HD))
                      : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    float mx = fmaxf(fmaxf(lv[0], lv[1]), fmaxf(lv[2], lv[3]));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xFFFFFFFFu, mx, o));
    if (lane == 0) red[wid] = mx;
    __syncthreads();
    float M = -INFINITY;
    for (int w = 0; w < nw; ++w) M = fmaxf(M, red[w]);
    float den = 0.f;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int j = tid + i * nt;
        const float w = lv[i] == -INFINITY ? 0.f : ex2f(lv[i] - M);
        if (j < n) w_all[j] = w;
        den += w;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) den += __shfl_xor_sync(0xFFFFFFFFu, den, o);
    __syncthreads();  // red[] read by all; w_all complete
    if (lane == 0) red[wid] = den;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int j = (tid >> 1) + i * hn;
        if (j < n) {
            const float w = w_all[j];
            acc.x = fmaf(w, ov[i].x, acc.x);
            acc.y = fmaf(w, ov[i].y, acc.y);
            acc.z = fmaf(w, ov[i].z, acc.z);
            acc.w = fmaf(w, ov[i].w, acc.w);
        }
    }
#pragma unroll
    for (int o = 16; o > 1; o >>= 1) {  // lanes of the same half
        acc.x += __shfl_xor_sync(0xFFFFFFFFu, acc.x, o);
        acc.y += __shfl_xor_sync(0xFFFFFFFFu, acc.y, o);
        acc.z += __shfl_xor_sync(0xFFFFFFFFu, acc.z, o);
        acc.w += __shfl_xor_sync(0xFFFFFFFFu, acc.w, o);
    }
    if (lane < 2) red4[wid][lane] = acc;
    __syncthreads();
    if (tid < 2) {
        float D = 0.f;
        float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int w = 0; w < nw; ++w) {
            D += red[w];
            a.x += red4[w][tid].x;
            a.y += red4[w][tid].y;
            a.z += red4[w][tid].z;
            a.w += red4[w][tid].w;
        }
        const float inv = D > 0.f ? 1.f / D : 0.f;
        T* out = static_cast<T*>(p.out) + static_cast<size_t>(kvh) * G * HD + c0 + 4 * tid;
        Vec<T>::store(out, a.x * inv);
        Vec<T>::store(out + 1, a.y * inv);
        Vec<T>::store(out + 2, a.z * inv);
        Vec<T>::store(out + 3, a.w * inv);
        if (tid == 0 && c0 % HD == 0 && p.lse)
            p.lse[kvh * G + h] = D > 0.f ? (M + __log2f(D)) * 0.69314718055994530942f : -INFINITY;
    }
    __syncthreads();  // shared scratch reused by the next slice
}

// Tail shared by both kernels: NS per-slot states (m, l in log2 units, unnormalised o) are in
// shared memory; merge them (R3), then write the output (one split) or this split's partial
// and run the in-kernel two-level split merge.
template <typename T, int HD, int G>
__device__ void finish_cta(const DecodeParams& p, const int kvh, const int split, const int NS, const float* sm_o,
                           const float* sm_ml, float* w_sh,
                           float* lse_sh, int* s_last) {
    __syncthreads();
    if (threadIdx.x < G) {
        const int h = threadIdx.x;
        float M = -INFINITY;
        for (int j = 0; j < NS; ++j) M = fmaxf(M, sm_ml[(j * G + h) * 2]);
        float den = 0.f;
        for (int j = 0; j < NS; ++j) {
            const float mj = sm_ml[(j * G + h) * 2];
            const float w = mj == -INFINITY ? 0.f : ex2f(mj - M);
            w_sh[j * G + h] = w;
            den += w * sm_ml[(j * G + h) * 2 + 1];
        }
        const float inv = den > 0.f ? 1.f / den : 0.f;
        for (int j = 0; j < NS; ++j) w_sh[j * G + h] *= inv;
        lse_sh[h] = den > 0.f ? M + __log2f(den) : -INFINITY;
    }
    __syncthreads();
    const bool single = p.n_split == 1;
    float* o1 = p.o1 + (static_cast<size_t>(kvh) * kMaxSplit + split) * G * HD;
    T* outp = static_cast<T*>(p.out) + static_cast<size_t>(kvh) * G * HD;
    for (int x = threadIdx.x; x < G * HD; x += blockDim.x) {
        const int h = x / HD;
        float acc = 0.f;
#pragma unroll 4
        for (int j = 0; j < NS; ++j) acc = fmaf(w_sh[j * G + h], sm_o[j * G * HD + x], acc);
        if (single)
            Vec<T>::store(outp + x, acc);
        else
            o1[x] = acc;
    }
    if (threadIdx.x < G) {
        if (single) {
            if (p.lse) p.lse[kvh * G + threadIdx.x] = lse_sh[threadIdx.x] * 0.69314718055994530942f;
        } else {
            p.l1[(static_cast<size_t>(kvh) * kMaxSplit + split) * G + threadIdx.x] = lse_sh[threadIdx.x];
        }
    }
    dstamp(2);
    if (single) return;
#if CDSP_DEC_MERGE
    {
        __threadfence();
        __syncthreads();
        if (threadIdx.x == 0) *s_last = atomicAdd(p.cnt2 + kvh, 1);
        __syncthreads();
        const int n = p.n_split, nsl = G * HD / 8;
        const int K = min(nsl, n), r = *s_last;
        if (r < n - K) return;
        if (threadIdx.x == 0) {  // wait for every split's partial
            const uint64_t t0 = ptx::globaltimer();
            for (;;) {
                int c;
                asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(c) : "l"(p.cnt2 + kvh) : "memory");
                if (c >= n) break;
                if (ptx::globaltimer() - t0 > 4000000000ull) __trap();
                __nanosleep(32);
            }
        }
        __syncthreads();
        dstamp(4);
        for (int sl = r - (n - K); sl < nsl; sl += K) merge_slice<T, HD, G>(p, kvh, sl);
        if (threadIdx.x == 0 && atomicAdd(p.cnt1 + kvh * kMaxGroups, 1) == K - 1) {
            p.cnt2[kvh] = 0;  // every merger has seen the full count: leave the workspace zeroed
            p.cnt1[kvh * kMaxGroups] = 0;
        }
        dstamp(6);
        return;
    }
#endif

    // ---- level 1: the last CTA of this group of kGroup splits merges them
    const int grp = split / kGroup;
    const int g0 = grp * kGroup, gn = min(kGroup, p.n_split - g0);
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
        const int prev = atomicAdd(p.cnt1 + kvh * kMaxGroups + grp, 1);
        *s_last = prev == gn - 1;
    }
    __syncthreads();
    if (!*s_last) return;
    dstamp(4);
    __threadfence();
    const bool final1 = p.n_groups == 1;
    merge_parts<T, HD, G>(p.o1 + (static_cast<size_t>(kvh) * kMaxSplit + g0) * G * HD,
                          p.l1 + (static_cast<size_t>(kvh) * kMaxSplit + g0) * G, gn,
                          p.o2 + (static_cast<size_t>(kvh) * kMaxGroups + grp) * G * HD,
                          p.l2 + (static_cast<size_t>(kvh) * kMaxGroups + grp) * G, final1 ? outp : nullptr,
                          final1 && p.lse ? p.lse + kvh * G : nullptr, w_sh, lse_sh);
    if (threadIdx.x == 0) p.cnt1[kvh * kMaxGroups + grp] = 0;  // leave the workspace zeroed
    dstamp(5);
    if (final1) return;

    // ---- level 2: the last group merger merges the groups
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
        const int prev = atomicAdd(p.cnt2 + kvh, 1);
        *s_last = prev == p.n_groups - 1;
    }
    __syncthreads();
    if (!*s_last) return;
    dstamp(6);
    __threadfence();
    merge_parts<T, HD, G>(p.o2 + static_cast<size_t>(kvh) * kMaxGroups * G * HD,
                          p.l2 + static_cast<size_t>(kvh) * kMaxGroups * G, p.n_groups, nullptr, nullptr, outp,
                          p.lse ? p.lse + kvh * G : nullptr, w_sh, lse_sh);
    if (threadIdx.x == 0) p.cnt2[kvh] = 0;
}

template <typename T, int HD, int G>
__global__ void __launch_bounds__(kThreads) decode_attn_kernel(const DecodeParams p) {
    constexpr int VEC = Vec<T>::N;          // elements per 16-byte vector
    constexpr int CPR = HD / VEC;           // vectors per K/V row (8, 16 or 32)
    constexpr int TPI = 32 / CPR;           // token rows per warp instruction
    constexpr int STEP = kNI * TPI;         // tokens per warp step
    constexpr int LOG_CPR = ilog2(CPR);
    static_assert(CPR >= kNI && CPR <= 32, "lane mapping");
    extern __shared__ float4 dsm[];
    float* sm = reinterpret_cast<float*>(dsm);
    float* sm_o = sm;                                   // [kWarps*TPI][G][HD]
    float* sm_ml = sm_o + kWarps * TPI * G * HD;         // [kWarps*TPI][G] x (m, l)
    float* w_sh = sm_ml + kWarps * TPI * G * 2;          // [max(kWarps*TPI, kMaxGroups)][G]
    float* lse_sh = w_sh + 32 * G;                       // [G]
    __shared__ int s_last;

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int c = lane % CPR, tsub = lane / CPR;
    const int kvh = blockIdx.y, split = blockIdx.x;
    const T* qp = static_cast<const T*>(p.q) + static_cast<size_t>(kvh) * G * HD + c * VEC;

    // q pre-scaled by sigma log2(e): scores come out in log2 units
    float q[G][VEC];
#pragma unroll
    for (int h = 0; h < G; ++h) {
        float f[VEC];
        Vec<T>::unpack(*reinterpret_cast<const uint4*>(qp + h * HD), f);
#pragma unroll
        for (int e = 0; e < VEC; ++e) q[h][e] = f[e] * p.scale_log2;
    }
    float m[G], l[G], o[G][VEC];
#pragma unroll
    for (int h = 0; h < G; ++h) {
        m[h] = -INFINITY;
        l[h] = 0.f;
#pragma unroll
        for (int e = 0; e < VEC; ++e) o[h][e] = 0.f;
    }

    const int64_t t0 = static_cast<int64_t>(split) * p.tok_per_split;
    const int64_t t1 = min(p.n_ctx, t0 + p.tok_per_split);
    const int64_t bmask = (int64_t{1} << p.b_shift) - 1;
    const size_t row = static_cast<size_t>(p.Hkv_t) * HD;  // elements per cache token row
    const T* kc = static_cast<const T*>(p.kc) + static_cast<size_t>(kvh) * HD + c * VEC;
    const T* vc = static_cast<const T*>(p.vc) + static_cast<size_t>(kvh) * HD + c * VEC;

    for (int64_t base = t0 + static_cast<int64_t>(warp) * STEP; base < t1; base += kWarps * STEP) {
        uint4 kr[kNI], vr[kNI];
        uint32_t valid = 0;
#pragma unroll
        for (int i = 0; i < kNI; ++i) {
            const int64_t tok = base + i * TPI + tsub;
            int64_t blk = -1;
            if (tok < t1) blk = __ldg(p.bt + (tok >> p.b_shift));
            if (blk >= 0 && blk < p.num_blocks) {
                const size_t off = static_cast<size_t>((blk << p.b_shift) | (tok & bmask)) * row;
                kr[i] = ld_stream(kc + off);
                vr[i] = ld_stream(vc + off);
                valid |= 1u << i;
            } else {
                kr[i] = make_uint4(0, 0, 0, 0);
                vr[i] = make_uint4(0, 0, 0, 0);
            }
        }
        // q . k for every (head, token): i outer so one token's K floats are live at a time
        float d[G][kNI];
#pragma unroll
        for (int i = 0; i < kNI; ++i) {
            float kf[VEC];
            Vec<T>::unpack(kr[i], kf);
#pragma unroll
            for (int h = 0; h < G; ++h) {
                float a = 0.f;
#pragma unroll
                for (int e = 0; e < VEC; ++e) a = fmaf(q[h][e], kf[e], a);
                d[h][i] = a;
            }
        }
#pragma unroll
        for (int h = 0; h < G; ++h) {
            // reduce-scatter over the CPR lanes of the row: the top 3 lane bits pick the token
#pragma unroll
            for (int lvl = 0; lvl < LOG_CPR; ++lvl) {
                const int lb = CPR >> (lvl + 1);
                const bool up = (lane & lb) != 0;
                if (lvl < 3) {
                    const int hn = kNI >> (lvl + 1);
#pragma unroll
                    for (int j = 0; j < hn; ++j) {
                        const float send = up ? d[h][j] : d[h][j + hn];
                        const float keep = up ? d[h][j + hn] : d[h][j];
                        d[h][j] = keep + __shfl_xor_sync(0xFFFFFFFFu, send, lb);
                    }
                } else {
                    d[h][0] += __shfl_xor_sync(0xFFFFFFFFu, d[h][0], lb);
                }
            }
            // gather the slot's kNI scores back; online softmax (log2 units), branch-free on -inf
            const float own = d[h][0];
            float mx = -INFINITY;
#pragma unroll
            for (int i = 0; i < kNI; ++i) {
                float si = __shfl_sync(0xFFFFFFFFu, own, tsub * CPR + (i << (LOG_CPR - 3)));
                si = ((valid >> i) & 1u) ? si : -INFINITY;
                d[h][i] = si;
                mx = fmaxf(mx, si);
            }
            const float mn = fmaxf(m[h], mx);
            const float mu = mn == -INFINITY ? 0.f : mn;
            const float alpha = ex2f(m[h] - mu);
            m[h] = mn;
            float ls = 0.f;
#pragma unroll
            for (int i = 0; i < kNI; ++i) {
                d[h][i] = ex2f(d[h][i] - mu);
                ls += d[h][i];
            }
            l[h] = l[h] * alpha + ls;
#pragma unroll
            for (int e = 0; e < VEC; ++e) o[h][e] *= alpha;
        }
        // P V: i outer so one token's V floats are live at a time
#pragma unroll
        for (int i = 0; i < kNI; ++i) {
            float vf[VEC];
            Vec<T>::unpack(vr[i], vf);
#pragma unroll
            for (int h = 0; h < G; ++h)
#pragma unroll
                for (int e = 0; e < VEC; ++e) o[h][e] = fmaf(d[h][i], vf[e], o[h][e]);
        }
    }

    // ---- CTA merge of the kWarps x TPI lane-group states
    const int slot = warp * TPI + tsub;
#pragma unroll
    for (int h = 0; h < G; ++h) {
#pragma unroll
        for (int e = 0; e < VEC; ++e) sm_o[(slot * G + h) * HD + c * VEC + e] = o[h][e];
        if (c == 0) {
            sm_ml[(slot * G + h) * 2] = m[h];
            sm_ml[(slot * G + h) * 2 + 1] = l[h];
        }
    }
    finish_cta<T, HD, G>(p, blockIdx.y, blockIdx.x, kWarps * TPI, sm_o, sm_ml, w_sh, lse_sh, &s_last);
}

// ---------------------------------------------------------------------------------------
// bf16: tensor-core decode.  The SIMT kernel above spends ~2000 issue slots per 16 tokens on
// dot products, unpacking and shuffles (ncu: 47% issue-busy at 2.3 TB/s, occupancy-starved at
// 183 registers), so it cannot reach the HBM rate.  Here each warp streams its own 16-token
// steps global -> shared memory with cp.async (3-stage ring per warp, 16-byte chunks
// XOR-swizzled by token so ldmatrix is conflict-free; out-of-range tokens zero-filled) and
// computes with mma.sync m16n8k16 (bf16 in, fp32 accumulate): S = Q K^T with the G query
// heads as rows 0..G-1 of M=16 (the rest zero), the accumulator re-packed in registers as P
// (the A operand of O += P V, V via ldmatrix.trans).  ~200 instructions per 16 tokens.  This is
// an HBM stream: one query row per head gives no M to fill a tcgen05 tile, so the legacy
// warp-level MMA is the right tool (its rate is far above the ~360 FLOP/clk/SM needed).
#ifndef CDSP_DEC_WARPS  // warps per CTA of the bf16 decode kernel (each streams its own token steps)
#define CDSP_DEC_WARPS 4
#endif
#ifndef CDSP_DEC_STAGES  // cp.async ring depth per warp (16-token K + V steps)
#define CDSP_DEC_STAGES 3
#endif
constexpr int kMmaWarps = CDSP_DEC_WARPS;
constexpr int kStages = CDSP_DEC_STAGES;

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, bool pred) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(pred ? 16 : 0)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(addr));
}
// D = A B + C for one m16n8k16 tile where A rows 8..15 are zero (a1 = a3 = 0): only the
// c0, c1 half (row g) is carried; the row g+8 half is discarded.
__device__ __forceinline__ void mma_top(float& c0, float& c1, uint32_t a0, uint32_t a2, uint32_t b0, uint32_t b1) {
    float d2, d3;
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%10,%10};"
        : "+f"(c0), "+f"(c1), "=f"(d2), "=f"(d3)
        : "r"(a0), "r"(0u), "r"(a2), "r"(0u), "r"(b0), "r"(b1), "f"(0.f));
}
__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
    const __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<const uint32_t*>(&v);
}

// PS: block size >= 16, so every (16-aligned) step lies in one page: one block-table lookup
template <int HD, int G, bool PS>
__global__ void __launch_bounds__(kMmaWarps * 32) decode_mma_kernel(const DecodeParams p) {
    constexpr int CH = HD / 8;                // 16-byte chunks per token row
    constexpr int ROWB = HD * 2;              // bytes per token row
    constexpr int TILE = 16 * ROWB;           // one 16-token K (or V) tile
    constexpr int NCP = 16 * CH / 32;         // chunks per lane per tile
    constexpr int KS = HD / 16;               // k-steps of S = Q K^T
    constexpr int ND = HD / 8;                // n-tiles of O
    extern __shared__ __align__(1024) uint8_t dsm_b[];
    __shared__ int s_last;
    dstamp(0);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g = lane >> 2, t = lane & 3;
    const int kvh = blockIdx.y, split = blockIdx.x;
    const uint32_t ring = static_cast<uint32_t>(__cvta_generic_to_shared(dsm_b)) + warp * kStages * 2 * TILE;
    // states for the CTA merge alias the rings (written after a CTA barrier)
    float* sm_o = reinterpret_cast<float*>(dsm_b);  // [kMmaWarps][G][HD]
    float* sm_ml = sm_o + kMmaWarps * G * HD;       // [kMmaWarps][G][2]
    float* w_sh = sm_ml + kMmaWarps * G * 2;        // [32][G]
    float* lse_sh = w_sh + 32 * G;
    static_assert((kMmaWarps * G * HD + kMmaWarps * G * 2 + 33 * G) * 4 <= kMmaWarps * kStages * 2 * TILE,
                  "merge state must fit in the rings");

    // Q as A fragments (rows = heads g < G, unscaled bf16; the scale is applied to S in fp32)
    uint32_t qa[KS][2];
    {
        const __nv_bfloat16* qp = static_cast<const __nv_bfloat16*>(p.q) + (static_cast<size_t>(kvh) * G + g) * HD;
#pragma unroll
        for (int kk = 0; kk < KS; ++kk) {
            qa[kk][0] = g < G ? *reinterpret_cast<const uint32_t*>(qp + 16 * kk + 2 * t) : 0u;
            qa[kk][1] = g < G ? *reinterpret_cast<const uint32_t*>(qp + 16 * kk + 2 * t + 8) : 0u;
        }
    }
    float o[ND][2];
#pragma unroll
    for (int nd = 0; nd < ND; ++nd) o[nd][0] = o[nd][1] = 0.f;
    float m = -INFINITY, l = 0.f;  // row g; l is this lane's partial row sum (quad-reduced at the end)

    const int64_t t0 = static_cast<int64_t>(split) * p.tok_per_split;
    const int64_t t1 = min(p.n_ctx, t0 + p.tok_per_split);
    const int64_t n_steps = (t1 - t0 + 15) / 16;
    const int64_t bmask = (int64_t{1} << p.b_shift) - 1;
    const size_t rowel = static_cast<size_t>(p.Hkv_t) * HD;
    const __nv_bfloat16* kc = static_cast<const __nv_bfloat16*>(p.kc) + static_cast<size_t>(kvh) * HD;
    const __nv_bfloat16* vc = static_cast<const __nv_bfloat16*>(p.vc) + static_cast<size_t>(kvh) * HD;

    // issue the copies of this warp's j-th step (tokens t0 + 16 (warp + j kMmaWarps) ..) into stage j % kStages
    auto issue = [&](int64_t j) {
        const int64_t base = t0 + 16 * (warp + j * kMmaWarps);
        const uint32_t sk = ring + static_cast<uint32_t>(j % kStages) * 2 * TILE, sv = sk + TILE;
        int64_t blk0 = -1;
        if (PS && base < t1) blk0 = __ldg(p.bt + (base >> p.b_shift));  // one page per step
#pragma unroll
        for (int i = 0; i < NCP; ++i) {
            const int id = i * 32 + lane, tok = id / CH, ch = id % CH;
            const int64_t pos = base + tok;
            int64_t blk = blk0;
            if (!PS) blk = pos < t1 ? __ldg(p.bt + (pos >> p.b_shift)) : -1;
            const bool ok = pos < t1 && blk >= 0 && blk < p.num_blocks;
            const size_t off = ok ? static_cast<size_t>((blk << p.b_shift) | (pos & bmask)) * rowel + ch * 8 : 0;
            const uint32_t so = static_cast<uint32_t>(tok * ROWB + ((ch ^ (tok & 7)) << 4));
            cp_async16(sk + so, kc + off, ok);
            cp_async16(sv + so, vc + off, ok);
        }
        cp_async_commit();
    };
    const int64_t my_steps = n_steps > warp ? (n_steps - warp + kMmaWarps - 1) / kMmaWarps : 0;
#pragma unroll
    for (int j = 0; j < kStages - 1; ++j) {
        if (j < my_steps) issue(j);
        else cp_async_commit();
    }
    for (int64_t j = 0; j < my_steps; ++j) {
        if (j + kStages - 1 < my_steps) issue(j + kStages - 1);
        else cp_async_commit();
        cp_async_wait<kStages - 1>();
        __syncwarp();
        const uint32_t sk = ring + static_cast<uint32_t>(j % kStages) * 2 * TILE, sv = sk + TILE;
        const int64_t base = t0 + 16 * (warp + j * kMmaWarps);
        // ---- S = Q K^T for 16 tokens (two n-tiles of 8)
        // (even / odd k-steps accumulate separately: four independent MMA chains, not two)
        float s[2][2] = {{0.f, 0.f}, {0.f, 0.f}}, s2[2][2] = {{0.f, 0.f}, {0.f, 0.f}};
#pragma unroll
        for (int kk = 0; kk < KS; kk += 2) {
#pragma unroll
            for (int nt = 0; nt < 2; ++nt) {
                // matrices i = 0..3: tokens 8nt + (lane & 7), chunk 2kk + i (lane >> 3)
                const int tok = 8 * nt + (lane & 7), ch = 2 * kk + (lane >> 3);
                uint32_t b0, b1, b2, b3;
                ldsm_x4(sk + tok * ROWB + ((ch ^ (tok & 7)) << 4), b0, b1, b2, b3);
                mma_top(s[nt][0], s[nt][1], qa[kk][0], qa[kk][1], b0, b1);
                mma_top(s2[nt][0], s2[nt][1], qa[kk + 1][0], qa[kk + 1][1], b2, b3);
            }
        }
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) {
            s[nt][0] += s2[nt][0];
            s[nt][1] += s2[nt][1];
        }
        // ---- online softmax on row g (log2 units); columns 8nt + 2t + e.  Tokens past the
        // split or on out-of-range pages were zero-filled: mask them.
        int64_t blk_step = 0;
        if (PS && base < t1) blk_step = __ldg(p.bt + (base >> p.b_shift));
        float mx = -INFINITY;
#pragma unroll
        for (int nt = 0; nt < 2; ++nt)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int64_t pos = base + 8 * nt + 2 * t + e;
                int64_t blk = blk_step;
                if (!PS && pos < t1) blk = __ldg(p.bt + (pos >> p.b_shift));
                const bool vis = pos < t1 && blk >= 0 && blk < p.num_blocks;
                s[nt][e] = vis ? s[nt][e] * p.scale_log2 : -INFINITY;
                mx = fmaxf(mx, s[nt][e]);
            }
        mx = fmaxf(mx, __shfl_xor_sync(0xFFFFFFFFu, mx, 1));
        mx = fmaxf(mx, __shfl_xor_sync(0xFFFFFFFFu, mx, 2));
        // lazy max: move only when the step's max exceeds the running one by > 8 (P <= 2^8)
        if (__any_sync(0xFFFFFFFFu, mx > m + 8.f)) {
            const float mn = fmaxf(m, mx);
            const float alpha = ex2f(m - mn);  // m = -inf: 0
            m = mn;
            l *= alpha;
#pragma unroll
            for (int nd = 0; nd < ND; ++nd) {
                o[nd][0] *= alpha;
                o[nd][1] *= alpha;
            }
        }
        const float mu = m == -INFINITY ? 0.f : m;
        float pr[2][2];
#pragma unroll
        for (int nt = 0; nt < 2; ++nt)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                pr[nt][e] = ex2f(s[nt][e] - mu);
                l += pr[nt][e];
            }
        // P as the A fragment of O += P V (k = the 16 tokens): a0 = tokens 2t.., a2 = 8 + 2t..
        const uint32_t pa0 = pack_bf16x2(pr[0][0], pr[0][1]), pa2 = pack_bf16x2(pr[1][0], pr[1][1]);
#pragma unroll
        for (int nd = 0; nd < ND; nd += 2) {
            // matrices: (tokens 0-7, chunk nd), (8-15, nd), (0-7, nd+1), (8-15, nd+1)
            const int tok = (lane & 7) + 8 * ((lane >> 3) & 1), ch = nd + (lane >> 4);
            uint32_t b0, b1, b2, b3;
            ldsm_x4_t(sv + tok * ROWB + ((ch ^ (tok & 7)) << 4), b0, b1, b2, b3);
            mma_top(o[nd][0], o[nd][1], pa0, pa2, b0, b1);
            mma_top(o[nd + 1][0], o[nd + 1][1], pa0, pa2, b2, b3);
        }
        __syncwarp();  // every lane is done with this stage before it is refilled
    }
    cp_async_wait<0>();
    l += __shfl_xor_sync(0xFFFFFFFFu, l, 1);
    l += __shfl_xor_sync(0xFFFFFFFFu, l, 2);

    // ---- per-warp state -> shared memory (slot = warp), then the common tail
    __syncthreads();  // all warps are done with their rings
    dstamp(1);
    if (g < G) {
#pragma unroll
        for (int nd = 0; nd < ND; ++nd) {
            sm_o[(warp * G + g) * HD + 8 * nd + 2 * t] = o[nd][0];
            sm_o[(warp * G + g) * HD + 8 * nd + 2 * t + 1] = o[nd][1];
        }
        if (t == 0) {
            sm_ml[(warp * G + g) * 2] = m;
            sm_ml[(warp * G + g) * 2 + 1] = l;
        }
    }
    finish_cta<__nv_bfloat16, HD, G>(p, blockIdx.y, blockIdx.x, kMmaWarps, sm_o, sm_ml, w_sh, lse_sh, &s_last);
    dstamp(3);
}

// ---------------------------------------------------------------------------------------
// bf16, block size >= 16: TMA-fed decode.  One producer thread streams the CTA's token range
// in 64-token stages (4 sub-tiles of 16 tokens = one page piece each: 128-byte-swizzled TMA
// boxes of 16 rows x 64 d of K and of V, pages looked up in the block table; a sub-tile past
// the range or on an out-of-range page is loaded from beyond the tensor, i.e. zero-filled)
// into an NST-deep ring of mbarrier-tracked stages; consumer warp w computes sub-tile w of
// every stage with mma.sync exactly as decode_mma_kernel does.  Against the per-warp cp.async
// rings: 8 TMA instructions per 64 tokens instead of 2 x 16 cp.async per lane per 16, and the
// bytes in flight per SM are set by the ring depth, not by the warps' issue.
#ifndef CDSP_DEC_TMA
#define CDSP_DEC_TMA 1
#endif
#ifndef CDSP_DEC_TMA_STAGES  // 64-token K + V stages per CTA (32 KB each at d = 128)
#define CDSP_DEC_TMA_STAGES 3
#endif
#ifndef CDSP_DEC_TMA_WARPS  // consumer warps per CTA (one 16-token sub-tile of each stage each)
#define CDSP_DEC_TMA_WARPS 4
#endif
constexpr int kTW = CDSP_DEC_TMA_WARPS;
#ifndef CDSP_DEC_NOCOMPUTE
#define CDSP_DEC_NOCOMPUTE 0
#endif
constexpr int kTStage = 16 * kTW;            // tokens per stage
constexpr int kTNst = CDSP_DEC_TMA_STAGES;

struct DecTmaArgs {
    CUtensorMap k, v;  // [num_blocks * B, Hkv_t, D], box 16 rows x 1 head x 64 d
    DecodeParams p;
    int64_t oob_row;   // a row coordinate past the tensor (zero-filled box)
};
// A batch of requests: a 1D grid over every request's (KV head, split) pairs back to back; CTA
// i belongs to request b with pre[b] <= i < pre[b + 1] (n_split_b = (pre[b + 1] - pre[b]) /
// Hkv_t splits of each of its KV heads), found by a binary search in kernel-parameter space.
constexpr int kMaxBatch = 1024;
struct DecTmaBatchArgs : DecTmaArgs {
    int32_t nb;
    int32_t pre[kMaxBatch + 1];
    int32_t ctx[kMaxBatch];
};

template <int HD>
struct TmaDecLayout {
    static constexpr int NH = HD / 64;                  // 64-d boxes per token row
    static constexpr int BOX = 16 * 128;                // 16 rows x 128 bytes
    static constexpr int SUB = NH * BOX;                // one 16-token sub-tile of K (or V)
    static constexpr int STAGE = 2 * kTW * SUB;         // K sub-tiles, then V sub-tiles
    static constexpr int RING = kTNst * STAGE;
    static constexpr int SMEM = RING + 1024;            // + alignment
};
template <int HD>
__device__ __forceinline__ uint32_t tdec_chunk(uint32_t sub, int tok, int ch) {  // 16-byte chunk ch of row tok
    return sub + static_cast<uint32_t>((ch >> 3) * TmaDecLayout<HD>::BOX + tok * 128 + (((ch & 7) ^ (tok & 7)) << 4));
}

template <int HD, int G, typename Args>
__global__ void __launch_bounds__((kTW + 1) * 32) decode_tma_kernel(const __grid_constant__ Args a) {
    using L = TmaDecLayout<HD>;
    constexpr int KS = HD / 16, ND = HD / 8;
    // virtual head vh = (request, KV head): the merge state, q, out and lse are indexed by it as
    // for one request of batch x Hkv_t heads; the cache by the request's table row and kvh.
    // One request: grid (split, KV head).  A batch (DecTmaBatchArgs): 1D grid, see there.
    DecodeParams p = a.p;
    int vh = blockIdx.y, split = blockIdx.x;
    if constexpr (sizeof(Args) == sizeof(DecTmaBatchArgs)) {
        const int i = static_cast<int>(blockIdx.x);
        int lo = 0, hi = a.nb;  // pre[lo] <= i < pre[hi]
        while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (a.pre[mid] <= i) lo = mid;
            else hi = mid;
        }
        const int ns = (a.pre[lo + 1] - a.pre[lo]) / p.Hkv_t;
        const int rr = i - a.pre[lo];
        p.n_ctx = a.ctx[lo];
        p.bt += static_cast<int64_t>(lo) * p.bt_stride;
        p.n_split = ns;
        p.n_groups = (ns + kGroup - 1) / kGroup;
        vh = lo * p.Hkv_t + rr / ns;
        split = rr % ns;
    }
    const int req = vh / p.Hkv_t;
    extern __shared__ uint8_t dsm_t[];
    __shared__ __align__(8) uint64_t full_b[kTNst], empty_b[kTNst];
    __shared__ int s_last;
    dstamp(0);
    uint8_t* sm = dsm_t + ((1024u - (static_cast<uint32_t>(__cvta_generic_to_shared(dsm_t)) & 1023u)) & 1023u);
    const uint32_t ring = static_cast<uint32_t>(__cvta_generic_to_shared(sm));
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int kvh = vh - req * p.Hkv_t;
    const int64_t t0 = static_cast<int64_t>(split) * p.tok_per_split;
    const int64_t t1 = min(p.n_ctx, t0 + p.tok_per_split);
    const int n_st = static_cast<int>((t1 - t0 + kTStage - 1) / kTStage);
    auto fb = [&](int i) { return static_cast<uint32_t>(__cvta_generic_to_shared(&full_b[i])); };
    auto eb = [&](int i) { return static_cast<uint32_t>(__cvta_generic_to_shared(&empty_b[i])); };
    if (threadIdx.x == 0) {
        for (int i = 0; i < kTNst; ++i) {
            ptx::mbar_init(fb(i), 1);
            ptx::mbar_init(eb(i), kTW);
        }
        ptx::fence_barrier_init();
    }
    __syncthreads();

    // states for the CTA merge alias the ring (written after the last stage is consumed)
    float* sm_o = reinterpret_cast<float*>(sm);     // [kTW][G][HD]
    float* sm_ml = sm_o + kTW * G * HD;             // [kTW][G][2]
    float* w_sh = sm_ml + kTW * G * 2;              // [32][G]
    float* lse_sh = w_sh + 32 * G;
    static_assert((kTW * G * HD + kTW * G * 2 + 33 * G) * 4 <= L::RING, "merge state must fit in the ring");

    const int g = lane >> 2, t = lane & 3;
    float o[ND][2];
#pragma unroll
    for (int nd = 0; nd < ND; ++nd) o[nd][0] = o[nd][1] = 0.f;
    float m = -INFINITY, l = 0.f;
    if (warp == kTW) {
        // ===== producer: one thread issues every TMA of the CTA's range
        if (lane == 0) {
            ptx::tma_prefetch_desc(&a.k);
            ptx::tma_prefetch_desc(&a.v);
            for (int j = 0; j < n_st; ++j) {
                const int st = j % kTNst;
                if (j >= kTNst) ptx::mbar_wait(eb(st), ((j / kTNst) - 1) & 1);
                ptx::mbar_expect_tx(fb(st), L::STAGE);
                const uint32_t sb = ring + static_cast<uint32_t>(st) * L::STAGE;
#pragma unroll
                for (int w = 0; w < kTW; ++w) {
                    const int64_t base = t0 + static_cast<int64_t>(j) * kTStage + 16 * w;
                    int64_t row = a.oob_row;
                    if (base < t1) {
                        const int64_t blk = __ldg(p.bt + (base >> p.b_shift));
                        if (blk >= 0 && blk < p.num_blocks) row = (blk << p.b_shift) | (base & ((int64_t{1} << p.b_shift) - 1));
                    }
#pragma unroll
                    for (int h = 0; h < L::NH; ++h) {
                        ptx::tma_load_3d(sb + w * L::SUB + h * L::BOX, &a.k, fb(st), 64 * h, kvh, static_cast<int>(row));
                        ptx::tma_load_3d(sb + (kTW + w) * L::SUB + h * L::BOX, &a.v, fb(st), 64 * h, kvh,
                                         static_cast<int>(row));
                    }
                }
            }
        }
        __syncwarp();
    } else {
        // ===== consumer warp w: sub-tile w of every stage
        uint32_t qa[KS][2];
        {
            const __nv_bfloat16* qp = static_cast<const __nv_bfloat16*>(p.q) + (static_cast<size_t>(vh) * G + g) * HD;
#pragma unroll
            for (int kk = 0; kk < KS; ++kk) {
                qa[kk][0] = g < G ? *reinterpret_cast<const uint32_t*>(qp + 16 * kk + 2 * t) : 0u;
                qa[kk][1] = g < G ? *reinterpret_cast<const uint32_t*>(qp + 16 * kk + 2 * t + 8) : 0u;
            }
        }
        for (int j = 0; j < n_st; ++j) {
            const int st = j % kTNst;
            const int64_t base = t0 + static_cast<int64_t>(j) * kTStage + 16 * warp;
            ptx::mbar_wait(fb(st), (j / kTNst) & 1);
            const uint32_t sk = ring + static_cast<uint32_t>(st) * L::STAGE + warp * L::SUB;
            const uint32_t sv = sk + kTW * L::SUB;
            if (!CDSP_DEC_NOCOMPUTE && base < t1) {  // (NOCOMPUTE: dev probe of the stream alone)
                int64_t blk = __ldg(p.bt + (base >> p.b_shift));
                const bool page_ok = blk >= 0 && blk < p.num_blocks;
                const int nvis = page_ok ? static_cast<int>((t1 - base < 16 ? t1 - base : int64_t{16})) : 0;
                if (nvis < 16 && page_ok) {
                    // rows past the range are real cache rows (maybe never written): zero their V
                    // so that P = 0 cannot meet a NaN
                    for (int x = lane; x < (16 - nvis) * (HD / 8); x += 32) {
                        const int tok = nvis + x / (HD / 8), ch = x % (HD / 8);
                        asm volatile("st.shared.v4.b32 [%0], {%1,%1,%1,%1};" ::"r"(tdec_chunk<HD>(sv, tok, ch)), "r"(0u)
                                     : "memory");
                    }
                    __syncwarp();
                }
                float s[2][2] = {{0.f, 0.f}, {0.f, 0.f}}, s2[2][2] = {{0.f, 0.f}, {0.f, 0.f}};
#pragma unroll
                for (int kk = 0; kk < KS; kk += 2) {
#pragma unroll
                    for (int nt = 0; nt < 2; ++nt) {
                        const int tok = 8 * nt + (lane & 7), ch = 2 * kk + (lane >> 3);
                        uint32_t b0, b1, b2, b3;
                        ldsm_x4(tdec_chunk<HD>(sk, tok, ch), b0, b1, b2, b3);
                        mma_top(s[nt][0], s[nt][1], qa[kk][0], qa[kk][1], b0, b1);
                        mma_top(s2[nt][0], s2[nt][1], qa[kk + 1][0], qa[kk + 1][1], b2, b3);
                    }
                }
                float mx = -INFINITY;
#pragma unroll
                for (int nt = 0; nt < 2; ++nt)
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        const int tk = 8 * nt + 2 * t + e;
                        const float sv2 = s[nt][e] + s2[nt][e];
                        s[nt][e] = tk < nvis ? sv2 * p.scale_log2 : -INFINITY;
                        mx = fmaxf(mx, s[nt][e]);
                    }
                mx = fmaxf(mx, __shfl_xor_sync(0xFFFFFFFFu, mx, 1));
                mx = fmaxf(mx, __shfl_xor_sync(0xFFFFFFFFu, mx, 2));
                if (__any_sync(0xFFFFFFFFu, mx > m + 8.f)) {  // lazy max (P <= 2^8), as decode_mma_kernel
                    const float mn = fmaxf(m, mx);
                    const float alpha = ex2f(m - mn);
                    m = mn;
                    l *= alpha;
#pragma unroll
                    for (int nd = 0; nd < ND; ++nd) {
                        o[nd][0] *= alpha;
                        o[nd][1] *= alpha;
                    }
                }
                const float mu = m == -INFINITY ? 0.f : m;
                float pr[2][2];
#pragma unroll
                for (int nt = 0; nt < 2; ++nt)
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        pr[nt][e] = ex2f(s[nt][e] - mu);
                        l += pr[nt][e];
                    }
                const uint32_t pa0 = pack_bf16x2(pr[0][0], pr[0][1]), pa2 = pack_bf16x2(pr[1][0], pr[1][1]);
#pragma unroll
                for (int nd = 0; nd < ND; nd += 2) {
                    const int tok = (lane & 7) + 8 * ((lane >> 3) & 1), ch = nd + (lane >> 4);
                    uint32_t b0, b1, b2, b3;
                    ldsm_x4_t(tdec_chunk<HD>(sv, tok, ch), b0, b1, b2, b3);
                    mma_top(o[nd][0], o[nd][1], pa0, pa2, b0, b1);
                    mma_top(o[nd + 1][0], o[nd + 1][1], pa0, pa2, b2, b3);
                }
                if (nvis < 16 && page_ok) ptx::fence_proxy_async_smem();  // generic writes before the next TMA
            }
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(eb(st));
        }
        l += __shfl_xor_sync(0xFFFFFFFFu, l, 1);
        l += __shfl_xor_sync(0xFFFFFFFFu, l, 2);
    }
    __syncthreads();  // every stage consumed: the ring is free for the merge state
    dstamp(1);
    if (warp < kTW && g < G) {
#pragma unroll
        for (int nd = 0; nd < ND; ++nd) {
            sm_o[(warp * G + g) * HD + 8 * nd + 2 * t] = o[nd][0];
            sm_o[(warp * G + g) * HD + 8 * nd + 2 * t + 1] = o[nd][1];
        }
        if (t == 0) {
            sm_ml[(warp * G + g) * 2] = m;
            sm_ml[(warp * G + g) * 2 + 1] = l;
        }
    }
    finish_cta<__nv_bfloat16, HD, G>(p, vh, split, kTW, sm_o, sm_ml, w_sh, lse_sh, &s_last);
    dstamp(3);
}

struct WsLayout {
    size_t cnt1, cnt2, l1, l2, o1, o2, total;
};
WsLayout ws_layout(int Hkv_t, int G, int D) {
    auto al = [](size_t x) { return (x + 255) / 256 * 256; };
    WsLayout w;
    w.cnt1 = 0;
    w.cnt2 = al(static_cast<size_t>(Hkv_t) * kMaxGroups * 4);
    w.l1 = w.cnt2 + al(static_cast<size_t>(Hkv_t) * 4);
    w.l2 = w.l1 + al(static_cast<size_t>(Hkv_t) * kMaxSplit * G * 4);
    w.o1 = w.l2 + al(static_cast<size_t>(Hkv_t) * kMaxGroups * G * 4);
    w.o2 = w.o1 + al(static_cast<size_t>(Hkv_t) * kMaxSplit * G * D * 4);
    w.total = w.o2 + al(static_cast<size_t>(Hkv_t) * kMaxGroups * G * D * 4);
    return w;
}

template <typename T, int HD, int G>
size_t simt_smem() {
    constexpr int VEC = 16 / static_cast<int>(sizeof(T));
    constexpr int TPI = 32 / (HD / VEC);
    return (static_cast<size_t>(kWarps) * TPI * G * HD + kWarps * TPI * G * 2 + 32 * G + G) * 4;
}
template <int HD>
constexpr size_t mma_smem() {
    return static_cast<size_t>(kMmaWarps) * kStages * 2 * 16 * HD * 2;
}

// The kernel a call runs: bf16 -> tensor-core kernel (TMA-fed for block size >= 16), f32 ->
// SIMT kernel.
struct Sel {
    const void* fn;
    int threads;
    size_t smem;
    int step;  // tokens per split granule
    bool tma;
};
template <int HD>
Sel select_tma(int G, bool batch) {
    using A = DecTmaArgs;
    using BA = DecTmaBatchArgs;
    const void* fn = G == 1 ? (batch ? reinterpret_cast<const void*>(decode_tma_kernel<HD, 1, BA>)
                                     : reinterpret_cast<const void*>(decode_tma_kernel<HD, 1, A>))
                   : G == 2 ? (batch ? reinterpret_cast<const void*>(decode_tma_kernel<HD, 2, BA>)
                                     : reinterpret_cast<const void*>(decode_tma_kernel<HD, 2, A>))
                   : G == 4 ? (batch ? reinterpret_cast<const void*>(decode_tma_kernel<HD, 4, BA>)
                                     : reinterpret_cast<const void*>(decode_tma_kernel<HD, 4, A>))
                            : (batch ? reinterpret_cast<const void*>(decode_tma_kernel<HD, 8, BA>)
                                     : reinterpret_cast<const void*>(decode_tma_kernel<HD, 8, A>));
    return {fn, (kTW + 1) * 32, static_cast<size_t>(TmaDecLayout<HD>::SMEM), kTStage, true};
}
template <typename T, int HD, int G>
Sel select_t(bool ps) {
    if constexpr (sizeof(T) == 2) {
        const void* fn = ps ? reinterpret_cast<const void*>(decode_mma_kernel<HD, G, true>)
                            : reinterpret_cast<const void*>(decode_mma_kernel<HD, G, false>);
        return {fn, kMmaWarps * 32, mma_smem<HD>(), 16, false};
    } else {
        constexpr int TPI = 32 / (HD / 4);
        return {reinterpret_cast<const void*>(decode_attn_kernel<T, HD, G>), kThreads, simt_smem<T, HD, G>(),
                kNI * TPI, false};
    }
}
template <typename T, int HD>
Sel select_g(int G, bool ps) {
    switch (G) {
        case 1: return select_t<T, HD, 1>(ps);
        case 2: return select_t<T, HD, 2>(ps);
        case 4: return select_t<T, HD, 4>(ps);
        default: return select_t<T, HD, 8>(ps);
    }
}
Sel select(int32_t dtype, int D, int G, bool ps, bool batch) {
    if ((CDSP_DEC_TMA || batch) && dtype == CDSP_BF16 && ps)
        return D == 128 ? select_tma<128>(G, batch) : select_tma<64>(G, batch);
    if (dtype == CDSP_BF16) return D == 128 ? select_g<__nv_bfloat16, 128>(G, ps) : select_g<__nv_bfloat16, 64>(G, ps);
    return D == 128 ? select_g<float, 128>(G, ps) : select_g<float, 64>(G, ps);
}

int sm_count() {
    static int n = 0;
    if (!n) {
        int dev = 0;
        if (cudaGetDevice(&dev) != cudaSuccess ||
            cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0)
            n = 148;
    }
    return n;
}

// resident CTAs per SM of a kernel (splits fill exactly one wave); sets the smem attribute once
int prepare(const Sel& k) {
    static const void* seen[64] = {};
    static int occ[64] = {};
    for (int i = 0; i < 64; ++i) {
        if (seen[i] == k.fn) return occ[i];
        if (!seen[i]) {
            int n = 0;
            cudaFuncSetAttribute(k.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(k.smem));
            if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k.fn, k.threads, k.smem) != cudaSuccess || n < 1)
                n = 1;
            seen[i] = k.fn;
            occ[i] = n;
            return n;
        }
    }
    return 1;
}

}  // namespace
}  // namespace cdsp

using namespace cdsp;

extern "C" {

cdsp_status cdsp_decode_workspace_bytes(int32_t hq_local, int32_t hkv_local, int32_t D, size_t* bytes) {
    CDSP_REQUIRE(bytes != nullptr, CDSP_ERR_INVALID, "bytes is NULL");
    CDSP_REQUIRE(hkv_local >= 1 && hq_local >= hkv_local && hq_local % hkv_local == 0, CDSP_ERR_SHAPE,
                 "Hq_t=%d must be a multiple of Hkv_t=%d", hq_local, hkv_local);
    CDSP_REQUIRE(D == 64 || D == 128, CDSP_ERR_SHAPE, "head dim %d not in {64,128}", D);
    *bytes = ws_layout(hkv_local, hq_local / hkv_local, D).total;
    return CDSP_OK;
}

}  // extern "C"

namespace {
// One decode step for `batch` requests (ctx_lens: host [batch]) or for one request of n_ctx
// (ctx_lens == NULL, batch == 1: cdsp_decode_attention).
cdsp_status decode_impl(const cdsp_tensor* q, const cdsp_decode_target* cache, int32_t t, int32_t hkv_local,
                        int32_t batch, const int32_t* ctx_lens, int64_t n_ctx, float softmax_scale, cdsp_tensor* out,
                        float* lse, void* workspace, size_t workspace_bytes, void* cuda_stream) {
    CDSP_REQUIRE(q && cache && out && workspace, CDSP_ERR_INVALID, "NULL argument");
    CDSP_REQUIRE(dtype_ok(q->dtype) && q->dtype == out->dtype, CDSP_ERR_DTYPE, "q/out dtype");
    CDSP_REQUIRE(q->ptr && out->ptr && (reinterpret_cast<uintptr_t>(q->ptr) & 15u) == 0 &&
                     (reinterpret_cast<uintptr_t>(out->ptr) & 15u) == 0,
                 CDSP_ERR_INVALID, "q/out must be non-NULL and 16-byte aligned");
    CDSP_REQUIRE(batch >= 1 && q->T == batch && out->T == batch && out->H == q->H && out->D == q->D,
                 CDSP_ERR_SHAPE, "q and out must be [%d, Hq_t, D]", batch);
    const int D = static_cast<int>(q->D);
    CDSP_REQUIRE(D == 64 || D == 128, CDSP_ERR_SHAPE, "head dim %d not in {64,128}", D);
    CDSP_REQUIRE(hkv_local >= 1 && q->H % hkv_local == 0, CDSP_ERR_SHAPE, "Hq_t=%lld not a multiple of Hkv_t=%d",
                 static_cast<long long>(q->H), hkv_local);
    const int G = static_cast<int>(q->H / hkv_local);
    CDSP_REQUIRE(G == 1 || G == 2 || G == 4 || G == 8, CDSP_ERR_UNSUPPORTED, "GQA group %d not in {1,2,4,8}", G);
    CDSP_REQUIRE(cache->tp >= 1 && cache->tp <= 8 && t >= 0 && t < cache->tp, CDSP_ERR_INVALID,
                 "decode rank %d of tp %d", t, cache->tp);
    CDSP_REQUIRE(cache->k_cache && cache->v_cache && cache->k_cache[t] && cache->v_cache[t] && cache->block_table,
                 CDSP_ERR_INVALID, "NULL cache pointer");
    const int B = cache->block_size;
    CDSP_REQUIRE(B >= 1 && B <= 4096 && (B & (B - 1)) == 0, CDSP_ERR_UNSUPPORTED,
                 "block size %d must be a power of two <= 4096", B);
    int64_t total_ctx = n_ctx;
    if (ctx_lens) {
        CDSP_REQUIRE(batch <= kMaxBatch, CDSP_ERR_CAPACITY, "batch %d exceeds %d", batch, kMaxBatch);
        n_ctx = 0;
        total_ctx = 0;
        for (int b = 0; b < batch; ++b) {
            CDSP_REQUIRE(ctx_lens[b] >= 1, CDSP_ERR_SHAPE, "ctx_lens[%d] = %d must be >= 1", b, ctx_lens[b]);
            n_ctx = std::max<int64_t>(n_ctx, ctx_lens[b]);
            total_ctx += ctx_lens[b];
        }
    }
    CDSP_REQUIRE(n_ctx >= 1, CDSP_ERR_SHAPE, "n_ctx must be >= 1");
    CDSP_REQUIRE(cache->n_table % batch == 0, CDSP_ERR_SHAPE, "block table of %lld entries is not %d rows",
                 static_cast<long long>(cache->n_table), batch);
    const int64_t row_len = cache->n_table / batch;  // block-table entries per request
    CDSP_REQUIRE(row_len * B >= n_ctx, CDSP_ERR_CAPACITY, "block table row covers %lld positions < n_ctx %lld",
                 static_cast<long long>(row_len * B), static_cast<long long>(n_ctx));
    const int vheads = batch * hkv_local;  // (request, KV head) pairs: the merge's heads
    CDSP_REQUIRE(vheads <= 65535, CDSP_ERR_CAPACITY, "batch x KV heads %d exceeds 65535", vheads);
    const WsLayout w = ws_layout(vheads, G, D);
    CDSP_REQUIRE(workspace_bytes >= w.total, CDSP_ERR_CAPACITY, "workspace %zu < %zu bytes", workspace_bytes,
                 w.total);
    CDSP_REQUIRE((reinterpret_cast<uintptr_t>(workspace) & 255u) == 0, CDSP_ERR_INVALID,
                 "workspace must be 256-byte aligned");

    DecodeParams p;
    std::memset(&p, 0, sizeof(p));
    p.q = q->ptr;
    p.kc = cache->k_cache[t];
    p.vc = cache->v_cache[t];
    p.bt = cache->block_table;
    p.bt_stride = row_len;
    p.num_blocks = cache->num_blocks;
    p.n_ctx = n_ctx;
    int sh = 0;
    while ((1 << sh) < B) ++sh;
    p.b_shift = sh;
    p.Hkv_t = hkv_local;
    const float scale = softmax_scale > 0.f ? softmax_scale : 1.0f / std::sqrt(static_cast<float>(D));
    p.scale_log2 = scale * 1.4426950408889634f;
    // split sizing: one wave of resident CTAs over all KV heads, whole warp-steps per split
    const Sel k = select(q->dtype, D, G, B >= 16, ctx_lens != nullptr);
    CDSP_REQUIRE(batch == 1 || k.tma, CDSP_ERR_UNSUPPORTED,
                 "a batch of requests needs the bf16 TMA kernel (block size >= 16)");
    const int occ = prepare(k);
    const int64_t steps = (n_ctx + k.step - 1) / k.step;
    // (rounded down: a split more per head than one wave holds would put a few CTAs in a second
    // wave, doubling the launch)
    int64_t want = static_cast<int64_t>(occ) * sm_count() / vheads;
    want = std::max<int64_t>(1, std::min<int64_t>(std::min<int64_t>(want, kMaxSplit), steps));
    int64_t steps_per = (steps + want - 1) / want;
    if (ctx_lens && total_ctx < static_cast<int64_t>(batch) * n_ctx) {
        // a batch of mixed lengths: the smallest split size whose splits, over all requests and
        // KV heads, fill at most one wave (each request gets ceil(steps_b / split) of them).  A few
        // slots are left free: a grid of exactly occupancy x SMs CTAs measured as two waves
        // (one CTA waiting makes its request's merge, and the launch, twice as long)
        const int64_t slots = static_cast<int64_t>(occ) * sm_count() - std::max(8, sm_count() / 16);
        int64_t sp = std::max<int64_t>(1, ((total_ctx + k.step - 1) / k.step * hkv_local + slots - 1) / slots);
        sp = std::max<int64_t>(sp, (steps + kMaxSplit - 1) / kMaxSplit);
        for (;; ++sp) {
            int64_t n = 0;
            for (int b = 0; b < batch; ++b) n += ((ctx_lens[b] + k.step - 1) / k.step + sp - 1) / sp;
            if (n * hkv_local <= slots || sp >= steps) break;
        }
        steps_per = sp;
    }
    p.tok_per_split = steps_per * k.step;
    p.n_split = static_cast<int>((n_ctx + p.tok_per_split - 1) / p.tok_per_split);
    p.n_groups = (p.n_split + kGroup - 1) / kGroup;
    char* ws = static_cast<char*>(workspace);
    p.cnt1 = reinterpret_cast<int*>(ws + w.cnt1);
    p.cnt2 = reinterpret_cast<int*>(ws + w.cnt2);
    p.l1 = reinterpret_cast<float*>(ws + w.l1);
    p.l2 = reinterpret_cast<float*>(ws + w.l2);
    p.o1 = reinterpret_cast<float*>(ws + w.o1);
    p.o2 = reinterpret_cast<float*>(ws + w.o2);
    p.out = out->ptr;
    p.lse = lse;
    cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
    if (k.tma) {
        const int64_t rows = cache->num_blocks * B;
        CDSP_REQUIRE(rows < (int64_t{1} << 31) - 1, CDSP_ERR_CAPACITY, "cache of %lld rows exceeds the TMA coordinate range",
                     static_cast<long long>(rows));
        DecTmaArgs ta;
        std::memset(&ta, 0, sizeof(ta));
        CDSP_CHECK_STATUS(make_tile_map(&ta.k, cache->k_cache[t], rows, hkv_local, D, 16));
        CDSP_CHECK_STATUS(make_tile_map(&ta.v, cache->v_cache[t], rows, hkv_local, D, 16));
        ta.p = p;
        ta.oob_row = rows;
        if (ctx_lens) {  // every request's (KV head, split) pairs back to back on a 1D grid
            static thread_local DecTmaBatchArgs tb;  // (8 KB: off the stack)
            static_cast<DecTmaArgs&>(tb) = ta;
            tb.nb = batch;
            tb.pre[0] = 0;
            for (int b = 0; b < batch; ++b) {
                tb.ctx[b] = ctx_lens[b];
                const int64_t ns = (ctx_lens[b] + p.tok_per_split - 1) / p.tok_per_split;
                tb.pre[b + 1] = tb.pre[b] + static_cast<int32_t>(ns * hkv_local);
            }
            void* bargs[] = {&tb};
            CDSP_CUDA(cudaLaunchKernel(k.fn, dim3(static_cast<unsigned>(tb.pre[batch])),
                                       dim3(static_cast<unsigned>(k.threads)), bargs, k.smem, st));
            return CDSP_OK;
        }
        void* targs[] = {&ta};
        CDSP_CUDA(cudaLaunchKernel(k.fn, dim3(static_cast<unsigned>(p.n_split), static_cast<unsigned>(vheads)),
                                   dim3(static_cast<unsigned>(k.threads)), targs, k.smem, st));
        return CDSP_OK;
    }
    void* args[] = {&p};
    CDSP_CUDA(cudaLaunchKernel(k.fn, dim3(static_cast<unsigned>(p.n_split), static_cast<unsigned>(hkv_local)),
                               dim3(static_cast<unsigned>(k.threads)), args, k.smem, st));
    return CDSP_OK;
}
}  // namespace

extern "C" {

cdsp_status cdsp_decode_attention(const cdsp_tensor* q, const cdsp_decode_target* cache, int32_t t,
                                  int32_t hkv_local, int64_t n_ctx, float softmax_scale, cdsp_tensor* out,
                                  float* lse, void* workspace, size_t workspace_bytes, void* cuda_stream) {
    return decode_impl(q, cache, t, hkv_local, 1, nullptr, n_ctx, softmax_scale, out, lse, workspace,
                       workspace_bytes, cuda_stream);
}

cdsp_status cdsp_decode_attention_batch(const cdsp_tensor* q, const cdsp_decode_target* cache, int32_t t,
                                        int32_t hkv_local, int32_t batch, const int32_t* ctx_lens, float softmax_scale,
                                        cdsp_tensor* out, float* lse, void* workspace, size_t workspace_bytes,
                                        void* cuda_stream) {
    CDSP_REQUIRE(ctx_lens != nullptr, CDSP_ERR_INVALID, "ctx_lens is NULL");
    return decode_impl(q, cache, t, hkv_local, batch, ctx_lens, 0, softmax_scale, out, lse, workspace,
                       workspace_bytes, cuda_stream);
}

#ifdef CDSP_DTRACE
CDSP_API cdsp_status cdsp_debug_decode_trace(unsigned long long* host4096x8) {
    CDSP_CUDA(cudaDeviceSynchronize());
    CDSP_CUDA(cudaMemcpyFromSymbol(host4096x8, g_dtrace, sizeof(unsigned long long) * 4096 * 8));
    return CDSP_OK;
}
#endif

}  // extern "C"
