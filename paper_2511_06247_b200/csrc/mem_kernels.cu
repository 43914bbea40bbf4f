// mem_kernels.cu — the HBM-bound kernels of the path:
//   K*3 n-way LSE merge (warp per row-head, shuffle-free: lanes own disjoint D slices)
//   K*4 zigzag gather / scatter and store append (16-byte vectorised row copies)
//   K*5 zigzag partition map
//   K*6 paged-KV scatter into decode caches
//   the peer barrier used by the ring (flags in peer memory over NVLink)
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "common.cuh"
#include "internal.h"

namespace cdsp {
namespace {

__device__ __forceinline__ uint64_t gtimer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// ------------------------------------------------------------------ K*3 LSE merge (R3)
struct MergeParams {
    int n;
    const float* parts[kMaxMerge];
    const float* lses[kMaxMerge];
    int64_t T;
    int H, D;
    void* out;
    int32_t out_dtype;
    float* lse;
};

// Loads that bypass L1 (every byte is read once) and streaming stores.
__device__ __forceinline__ float4 ld_stream4(const float* p) {
    float4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "l"(p));
    return v;
}
__device__ __forceinline__ float2 ld_stream2(const float* p) {
    float2 v;
    asm volatile("ld.global.nc.L1::no_allocate.v2.f32 {%0,%1}, [%2];" : "=f"(v.x), "=f"(v.y) : "l"(p));
    return v;
}

// Warp per (token, head) row: lane owns PER = D/32 contiguous elements of the row in every part.
// All of a row's loads — the n LSEs and the n partial slices — are issued before any is used
// (one memory round trip per row), and each warp walks RPI rows per iteration (grid-stride) so
// enough bytes are in flight at small n.  A part whose lse is -inf contributes nothing and its
// O is never multiplied in (R16: it may be unwritten).
template <int D, int NP, int RPI>
__global__ void __launch_bounds__(256) lse_merge_kernel(const MergeParams p) {
    constexpr int PER = D / 32;  // elements per lane (2 or 4)
    const int lane = threadIdx.x & 31;
    const int64_t rows = p.T * p.H;
    const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
    for (int64_t g0 = ((static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5) * RPI; g0 < rows;
         g0 += nwarps * RPI) {
        float a[RPI][NP];
        float x[RPI][NP][PER];
#pragma unroll
        for (int rr = 0; rr < RPI; ++rr) {
            const int64_t gw = g0 + rr;
            const bool ok = gw < rows;
            const int64_t t = ok ? gw / p.H : 0;
            const int h = ok ? static_cast<int>(gw % p.H) : 0;
            const size_t li = static_cast<size_t>(h) * p.T + t;
            const size_t base = static_cast<size_t>(ok ? gw : 0) * D + lane * PER;
#pragma unroll
            for (int i = 0; i < NP; ++i) {
                a[rr][i] = -INFINITY;
                if (ok && i < p.n) {
                    a[rr][i] = p.lses[i][li];
                    if constexpr (PER == 4) {
                        const float4 v = ld_stream4(p.parts[i] + base);
                        x[rr][i][0] = v.x;
                        x[rr][i][1] = v.y;
                        x[rr][i][2] = v.z;
                        x[rr][i][3] = v.w;
                    } else {
                        const float2 v = ld_stream2(p.parts[i] + base);
                        x[rr][i][0] = v.x;
                        x[rr][i][1] = v.y;
                    }
                }
            }
        }
#pragma unroll
        for (int rr = 0; rr < RPI; ++rr) {
            const int64_t gw = g0 + rr;
            if (gw >= rows) break;
            float M = -INFINITY;
#pragma unroll
            for (int i = 0; i < NP; ++i) M = fmaxf(M, a[rr][i]);
            float acc[PER];
#pragma unroll
            for (int e = 0; e < PER; ++e) acc[e] = 0.f;
            float den = 0.f;
            if (M != -INFINITY) {
#pragma unroll
                for (int i = 0; i < NP; ++i) {
                    const bool use = a[rr][i] != -INFINITY;
                    const float w = use ? __expf(a[rr][i] - M) : 0.f;
                    den += w;
#pragma unroll
                    for (int e = 0; e < PER; ++e) acc[e] = use ? fmaf(w, x[rr][i][e], acc[e]) : acc[e];
                }
            }
            const float inv = den > 0.f ? 1.0f / den : 0.f;
            const size_t ob = static_cast<size_t>(gw) * D + lane * PER;
            if (p.out_dtype == CDSP_F32) {
                float* o = static_cast<float*>(p.out) + ob;
                if constexpr (PER == 4)
                    __stcs(reinterpret_cast<float4*>(o), make_float4(acc[0] * inv, acc[1] * inv, acc[2] * inv, acc[3] * inv));
                else
                    __stcs(reinterpret_cast<float2*>(o), make_float2(acc[0] * inv, acc[1] * inv));
            } else {
                __nv_bfloat16* o = static_cast<__nv_bfloat16*>(p.out) + ob;
                if constexpr (PER == 4) {
                    const __nv_bfloat162 b0 = __floats2bfloat162_rn(acc[0] * inv, acc[1] * inv);
                    const __nv_bfloat162 b1 = __floats2bfloat162_rn(acc[2] * inv, acc[3] * inv);
                    uint2 u;
                    u.x = *reinterpret_cast<const uint32_t*>(&b0);
                    u.y = *reinterpret_cast<const uint32_t*>(&b1);
                    __stcs(reinterpret_cast<uint2*>(o), u);
                } else {
                    *reinterpret_cast<__nv_bfloat162*>(o) = __floats2bfloat162_rn(acc[0] * inv, acc[1] * inv);
                }
            }
            if (p.lse && lane == 0) {
                const int64_t t = gw / p.H;
                const int h = static_cast<int>(gw % p.H);
                p.lse[static_cast<size_t>(h) * p.T + t] = (M == -INFINITY) ? -INFINITY : M + __logf(den);
            }
        }
    }
}

// ------------------------------------------------------------------ K*4 row copies
struct RowCopyParams {
    RowCopy seg[2];
    int n_segs;
    int64_t row_vec;  // 16-byte vectors per row
    int64_t total;    // vectors over all segments
    int64_t seg0_vec;
};

// Warp per row (grid-stride over the rows of both segments; no per-vector division): lane
// copies 16-byte vectors lane, lane + 32, ... of the row, four loads in flight before the stores.
__global__ void __launch_bounds__(256) row_copy_kernel(const RowCopyParams p) {
    const int lane = threadIdx.x & 31;
    const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
    const int64_t rows0 = p.seg[0].n_rows, rows = rows0 + (p.n_segs > 1 ? p.seg[1].n_rows : 0);
    const int rv = static_cast<int>(p.row_vec);
    for (int64_t w = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; w < rows; w += nwarps) {
        const bool s1 = w >= rows0;
        const RowCopy& sg = s1 ? p.seg[1] : p.seg[0];
        const int64_t r = s1 ? w - rows0 : w;
        const uint4* src = static_cast<const uint4*>(sg.src) + (sg.src_row0 + r * sg.src_stride) * p.row_vec;
        uint4* dst = static_cast<uint4*>(sg.dst) + (sg.dst_row0 + r * sg.dst_stride) * p.row_vec;
        for (int c0 = lane; c0 < rv; c0 += 128) {
            uint4 v[4];
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (c0 + 32 * u < rv) v[u] = __ldcs(src + c0 + 32 * u);
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (c0 + 32 * u < rv) __stcs(dst + c0 + 32 * u, v[u]);
        }
    }
}

__global__ void __launch_bounds__(256) store_append_kernel(const AppendArgs a) {
    const int64_t row_vec = a.row_bytes / 16;
    const int64_t total = a.n_rows * row_vec;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total; i += stride) {
        static_cast<uint4*>(a.k_dst)[i] = __ldg(static_cast<const uint4*>(a.k_src) + i);
        static_cast<uint4*>(a.v_dst)[i] = __ldg(static_cast<const uint4*>(a.v_src) + i);
        if (i < a.n_rows)
            a.pos_dst[i] = static_cast<int32_t>(i < a.len0 ? a.pos0 + i * a.pos_stride
                                                           : a.pos1 + (i - a.len0) * a.pos_stride);
    }
}

__global__ void fill_positions_kernel(int32_t* dst, int64_t n, int64_t len0, int64_t pos0, int64_t pos1,
                                      int64_t pst) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) dst[i] = static_cast<int32_t>(i < len0 ? pos0 + i * pst : pos1 + (i - len0) * pst);
}

// ------------------------------------------------------------------ K*5 zigzag map
__global__ void zigzag_map_kernel(int64_t L, int s, int64_t m, int32_t* tok_rank, int32_t* tok_slot) {
    const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= L) return;
    const int64_t shard = t / m, off = t - shard * m;
    const bool first = shard < s;
    if (tok_rank) tok_rank[t] = static_cast<int32_t>(first ? shard : 2 * s - 1 - shard);
    if (tok_slot) tok_slot[t] = static_cast<int32_t>(first ? off : m + off);
}

// ------------------------------------------------------------------ K*6 paged scatter (R15)
// One warp per (token, K|V) row: the token's position and physical block are resolved once;
// the row [Hkv, D] splits into tp contiguous slices (one per decode TP rank), each copied to a
// contiguous slot [blk][p % B][Hkv/tp][D] of that rank's cache in 16-byte vectors.
// Grid-stride over (token, K|V) rows, one warp per row; each lane keeps 4 16-byte vectors in
// flight.
__global__ void __launch_bounds__(512) paged_scatter_kernel(const PagedArgs a) {
    const int wpb = blockDim.x >> 5;
    const int64_t nw = static_cast<int64_t>(gridDim.x) * wpb;
    const int lane = threadIdx.x & 31;
    const int seg_vec = a.seg_vec;                  // 16-byte vectors per TP slice (Hkv/tp heads)
    const int row_vec = seg_vec * a.tp;             // per token row
    for (int64_t w = static_cast<int64_t>(blockIdx.x) * wpb + (threadIdx.x >> 5); w < 2 * a.n_tok; w += nw) {
        const int which = w >= a.n_tok;  // 0: K, 1: V
        const int64_t tok = which ? w - a.n_tok : w;
        const int64_t pos = tok < a.len0 ? a.pos0 + tok * a.pos_stride : a.pos1 + (tok - a.len0) * a.pos_stride;
        const int64_t lb = pos / a.block_size;
        const int32_t blk = lb < a.n_table ? __ldg(a.block_table + lb) : -1;
        if (blk < 0 || blk >= a.num_blocks) {
            if (lane == 0 && which == 0) atomicAdd(a.bad_count, 1ull);
            continue;
        }
        const int64_t slot = static_cast<int64_t>(blk) * a.block_size + pos % a.block_size;
        const uint4* src = static_cast<const uint4*>(which ? a.v : a.k) + tok * row_vec;
        for (int c0 = 0; c0 < row_vec; c0 += 128) {
            uint4 x[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int c = c0 + 32 * u + lane;
                if (c < row_vec) x[u] = __ldg(src + c);
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int c = c0 + 32 * u + lane;
                if (c < row_vec) {
                    const int t = a.seg_shift >= 0 ? (c >> a.seg_shift) : c / seg_vec;
                    const int cl = c - t * seg_vec;
                    uint4* dst = static_cast<uint4*>(which ? a.v_cache[t] : a.k_cache[t]) + slot * seg_vec + cl;
                    *dst = x[u];
                }
            }
        }
    }
}

// ------------------------------------------------------------------ peer barrier
__global__ void peer_barrier_kernel(const BarrierArgs a) {
    const int j = threadIdx.x;
    if (j >= a.n) return;
    __threadfence_system();  // this stream's prior writes before the signal
    if (a.remote[j]) atomicAdd_system(a.remote[j], 1ull);  // NULL: wait only
    const uint64_t t0 = gtimer();
    while (true) {
        unsigned long long v;
        asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(a.local[j]) : "memory");
        if (v >= a.target[j]) break;
        if (gtimer() - t0 > 8000000000ull) {  // 8 s: a peer never arrived
            atomicExch(a.err, 1);
            break;
        }
        __nanosleep(64);
    }
    __threadfence_system();
}

int sm_count_dev() {
    static int n[64] = {};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
    if (n[dev] == 0 && cudaDeviceGetAttribute(&n[dev], cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) n[dev] = 148;
    return n[dev];
}

unsigned grid_for(int64_t work, int per_block = 256) {
    int64_t b = (work + per_block - 1) / per_block;
    const int64_t cap = 148 * 16;
    if (b > cap) b = cap;
    if (b < 1) b = 1;
    return static_cast<unsigned>(b);
}

}  // namespace

cdsp_status launch_lse_merge(int n, const float* const* parts, const float* const* lses, int64_t T, int H, int D,
                             void* out, int32_t out_dtype, float* lse, cudaStream_t st) {
    CDSP_REQUIRE(n >= 1 && n <= kMaxMerge, CDSP_ERR_INVALID, "merge count %d not in [1,%d]", n, kMaxMerge);
    MergeParams p;
    p.n = n;
    for (int i = 0; i < kMaxMerge; ++i) {
        p.parts[i] = i < n ? parts[i] : nullptr;
        p.lses[i] = i < n ? lses[i] : nullptr;
    }
    p.T = T;
    p.H = H;
    p.D = D;
    p.out = out;
    p.out_dtype = out_dtype;
    p.lse = lse;
    const int64_t warps = T * H;
    if (warps == 0) return CDSP_OK;
    CDSP_REQUIRE(D == 64 || D == 128, CDSP_ERR_SHAPE, "head dim %d not supported", D);
    // grid-stride: 8 CTAs of 8 warps per SM, each warp 1-2 rows per iteration
    const int64_t need = (warps + 1) / 2;
    const int64_t cap = static_cast<int64_t>(sm_count_dev()) * 8 * 8;
    const unsigned blocks = static_cast<unsigned>(((need < cap ? need : cap) + 7) / 8);
#define CDSP_MERGE_LAUNCH(DD, NP, RPI) lse_merge_kernel<DD, NP, RPI><<<blocks, 256, 0, st>>>(p)
    if (D == 128) {
        if (n <= 2) CDSP_MERGE_LAUNCH(128, 2, 2);
        else if (n <= 4) CDSP_MERGE_LAUNCH(128, 4, 2);
        else if (n <= 8) CDSP_MERGE_LAUNCH(128, 8, 1);
        else CDSP_MERGE_LAUNCH(128, 16, 1);
    } else {
        if (n <= 2) CDSP_MERGE_LAUNCH(64, 2, 2);
        else if (n <= 4) CDSP_MERGE_LAUNCH(64, 4, 2);
        else if (n <= 8) CDSP_MERGE_LAUNCH(64, 8, 2);
        else CDSP_MERGE_LAUNCH(64, 16, 1);
    }
#undef CDSP_MERGE_LAUNCH
    CDSP_CUDA(cudaGetLastError());
    return CDSP_OK;
}

cdsp_status launch_row_copy(const RowCopy* segs, int n_segs, int64_t row_bytes, cudaStream_t st) {
    CDSP_REQUIRE(n_segs >= 1 && n_segs <= 2, CDSP_ERR_INVALID, "row copy: 1 or 2 segments");
    CDSP_REQUIRE(row_bytes % 16 == 0, CDSP_ERR_SHAPE, "row bytes %lld not a multiple of 16",
                 static_cast<long long>(row_bytes));
    RowCopyParams p;
    p.n_segs = n_segs;
    p.row_vec = row_bytes / 16;
    p.seg[0] = segs[0];
    p.seg[1] = n_segs > 1 ? segs[1] : RowCopy{nullptr, nullptr, 0, 0, 0, 1, 1};
    p.seg0_vec = segs[0].n_rows * p.row_vec;
    p.total = p.seg0_vec + (n_segs > 1 ? segs[1].n_rows * p.row_vec : 0);
    if (p.total == 0) return CDSP_OK;
    const int64_t rows = segs[0].n_rows + (n_segs > 1 ? segs[1].n_rows : 0);
    const int64_t cap = static_cast<int64_t>(sm_count_dev()) * 8;  // 8 CTAs x 8 warps per SM
    const int64_t blocks = (rows + 7) / 8 < cap ? (rows + 7) / 8 : cap;
    row_copy_kernel<<<static_cast<unsigned>(blocks), 256, 0, st>>>(p);
    CDSP_CUDA(cudaGetLastError());
    return CDSP_OK;
}

cdsp_status launch_store_append(const AppendArgs& a, cudaStream_t st) {
    CDSP_REQUIRE(a.row_bytes % 16 == 0, CDSP_ERR_SHAPE, "row bytes not a multiple of 16");
    const int64_t work = a.n_rows * (a.row_bytes / 16);
    if (a.n_rows == 0) return CDSP_OK;
    store_append_kernel<<<grid_for(work > a.n_rows ? work : a.n_rows), 256, 0, st>>>(a);
    CDSP_CUDA(cudaGetLastError());
    return CDSP_OK;
}

cdsp_status launch_fill_positions(int32_t* dst, int64_t n, int64_t len0, int64_t pos0, int64_t pos1, int64_t pst,
                                  cudaStream_t st) {
    if (n == 0) return CDSP_OK;
    fill_positions_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(dst, n, len0, pos0, pos1, pst);
    CDSP_CUDA(cudaGetLastError());
    return CDSP_OK;
}

cdsp_status launch_zigzag_map(int64_t L, int s, int32_t* tok_rank, int32_t* tok_slot, cudaStream_t st) {
    if (L == 0) return CDSP_OK;
    const int64_t m = L / (2 * s);
    const int64_t blocks = (L + 255) / 256;
    zigzag_map_kernel<<<static_cast<unsigned>(blocks), 256, 0, st>>>(L, s, m, tok_rank, tok_slot);
    CDSP_CUDA(cudaGetLastError());
    return CDSP_OK;
}

cdsp_status launch_paged_scatter(const PagedArgs& a_in, cudaStream_t st) {
    PagedArgs a = a_in;
    CDSP_REQUIRE((a.D * a.esize) % 16 == 0, CDSP_ERR_SHAPE, "head row not a multiple of 16 bytes");
    a.seg_vec = (a.Hkv / a.tp) * a.D * a.esize / 16;
    a.seg_shift = -1;
    for (int sh = 0; sh < 30; ++sh)
        if ((1 << sh) == a.seg_vec) a.seg_shift = sh;
    const int64_t rows = 2 * a.n_tok;  // one warp per (token, K|V)
    if (rows == 0) return CDSP_OK;
    // CTAs of 16 warps, one warp per row.  CDSP_SCATTER_CTAS caps the grid (measurement control):
    // confining the scatter to 8-32 SMs beside the attention lengthened the bench step (the
    // scatter then outlasts the attention: 6.5 -> 6.8-7.9 ms), so the default is uncapped.
    static const int64_t cap = [] {
        const char* e = getenv("CDSP_SCATTER_CTAS");
        const long v = e ? strtol(e, nullptr, 10) : 0;
        return static_cast<int64_t>(v > 0 ? v : (1ll << 30));
    }();
    int64_t blocks = (rows + 15) / 16;
    if (blocks > cap) blocks = cap;
    paged_scatter_kernel<<<static_cast<unsigned>(blocks), 512, 0, st>>>(a);
    CDSP_CUDA(cudaGetLastError());
    return CDSP_OK;
}

cdsp_status launch_peer_barrier(const BarrierArgs& a, cudaStream_t st) {
    if (a.n == 0) return CDSP_OK;
    peer_barrier_kernel<<<1, 32, 0, st>>>(a);
    CDSP_CUDA(cudaGetLastError());
    return CDSP_OK;
}

}  // namespace cdsp
