// attn_tc.cu — K*1: bf16 block attention for one ring step on sm_100a tensor cores.
//
// Computes, for a query shard and one KV block (history + a current-chunk shard), exact
// softmax attention under the position mask of attn_common.cuh, and writes or LSE-merges
// the result (cdsp_attn_mode).  This is the per-step compute of ring attention
// (§2.3: each instance "interact[s] local query tensors with full key-value
// tensors"), extended to historical tokens as Tetris does (§6: "we extend Flash
// Attention [7] to support zigzag ring attention for historical tokens").
//
// B200 design (not the paper's A100 FlashAttention-2):
//  * one CTA = two 128-row query tiles sharing one KV head (two heads of a GQA group on the
//    same rows, or two adjacent row tiles of one MHA head); 12 warps:
//      warp 0  TMA producer (Q once, K/V 128-row tiles through a 2-stage ring each)
//      warp 1  TMEM allocator + single-thread tcgen05.mma issuer
//      warps 4-7 / 8-11  softmax + epilogue of query tile 0 / 1 (thread = row = TMEM lane)
//  * TMEM (512 cols): O0 [0,128) O1 [128,256) S0 [256,384) S1 [384,512); P (bf16) is
//    written over its S tile and fed to the PV MMA straight from TMEM (A operand).
//  * MMA order per KV tile j:  PV0(j), S0(j+1), PV1(j), S1(j+1) — the tensor core works on
//    one tile while the other tile's softmax runs.  A commit after S_t(j+1) also covers
//    PV_t(j), so softmax may rescale O_t in TMEM when it sees S_t(j+1).
//  * lazy rescaling: the running max only moves when it grows by > 8 (log2 units).
//  * masks from segment descriptors: empty tiles are skipped, full tiles run mask-free,
//    only diagonal / ragged tiles evaluate per-element positions.
#include <cuda.h>
#include <cuda_bf16.h>

#include "attn_common.cuh"
#include "common.cuh"
#include "internal.h"
#include "ptx.cuh"

namespace cdsp {
using namespace ptx;

namespace {

constexpr int kThreads = 384;
constexpr int BM = 128;  // query rows per tile (TMEM lanes)
constexpr int BN = 128;  // KV rows per tile
constexpr int kBoxBytes = 128 * 128;  // 128 rows x 64 bf16 (one 128-byte swizzle row each)

template <int HD>
struct Layout {
    static constexpr int NBOX = HD / 64;
    static constexpr int TILE = kBoxBytes * NBOX;  // one 128-row tile of Q, K or V
    static constexpr int KST = 2, VST = 2;
    static constexpr int OFF_Q = 0;
    static constexpr int OFF_K = OFF_Q + 2 * TILE;
    static constexpr int OFF_V = OFF_K + KST * TILE;
    static constexpr int OFF_BAR = OFF_V + VST * TILE;
    // q_full, k_full[KST], k_empty[KST], v_full[VST], v_empty[VST], s_full[2], p_full[2], o_full[2]
    static constexpr int B_Q = 0, B_KF = 1, B_KE = B_KF + KST, B_VF = B_KE + KST, B_VE = B_VF + VST,
                         B_S = B_VE + VST, B_P = B_S + 2, B_O = B_P + 2, NBAR = B_O + 2;
    static constexpr int OFF_TMEM_SLOT = OFF_BAR + NBAR * 8;
    static constexpr int SMEM = OFF_TMEM_SLOT + 16 + 1024;  // + alignment slack
};

constexpr uint32_t COL_O0 = 0, COL_O1 = 128, COL_S0 = 256, COL_S1 = 384;

struct TcParams {
    cdsp_segments seg;
    int Hq, Hkv, g, pair_heads, n_rb, n_hg;
    float scale_log2;
    int mode;
    float* o_acc;
    float* lse_acc;
    __nv_bfloat16* out;
    float* lse;
};

__device__ __forceinline__ void setmaxnreg_dec88() { asm volatile("setmaxnreg.dec.sync.aligned.u32 88;"); }
__device__ __forceinline__ void setmaxnreg_inc208() { asm volatile("setmaxnreg.inc.sync.aligned.u32 208;"); }

template <int HD>
__global__ void __launch_bounds__(kThreads, 1)
    attn_tc_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                   const __grid_constant__ CUtensorMap tm_v, const TcParams p) {
    using L = Layout<HD>;
    extern __shared__ uint8_t smem_raw[];
    // 1024-byte alignment for the 128B-swizzle atoms
    const uint32_t raw_addr = smem_u32(smem_raw);
    uint8_t* smem = smem_raw + ((1024u - (raw_addr & 1023u)) & 1023u);
    const uint32_t sbase = smem_u32(smem);
    const uint32_t sQ = sbase + L::OFF_Q, sK = sbase + L::OFF_K, sV = sbase + L::OFF_V;
    const uint32_t bar0 = sbase + L::OFF_BAR;
    auto bar = [&](int i) { return bar0 + 8u * static_cast<uint32_t>(i); };
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + L::OFF_TMEM_SLOT);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const cdsp_segments& sg = p.seg;

    // ---- work unit (heavy row blocks first: causal work grows with the row index)
    const int bid = blockIdx.x;
    const int rb = p.n_rb - 1 - bid / p.n_hg;
    const int hg = bid % p.n_hg;
    // (scalars, not arrays: tile index t is a runtime value and arrays would go to local memory)
    const int64_t row0_0 = p.pair_heads ? static_cast<int64_t>(rb) * BM : static_cast<int64_t>(rb) * 2 * BM;
    const int64_t row0_1 = p.pair_heads ? row0_0 : row0_0 + BM;
    const int head_0 = p.pair_heads ? 2 * hg : hg;
    const int head_1 = p.pair_heads ? 2 * hg + 1 : hg;
    const int kvh = head_0 / p.g;
    int64_t qlo_0, qhi_0, qlo_1, qhi_1;
    bool qany_0, qany_1;
    seg_qrange(sg, row0_0, row0_0 + BM, qlo_0, qhi_0, qany_0);
    seg_qrange(sg, row0_1, row0_1 + BM, qlo_1, qhi_1, qany_1);
    const int n_kv_tiles = static_cast<int>((sg.nkv + BN - 1) / BN);
    auto kind_of = [&](int t, int j) {
        const int64_t c0 = static_cast<int64_t>(j) * BN;
        return t == 0 ? seg_tile_kind(sg, qany_0, qlo_0, qhi_0, c0, BN) : seg_tile_kind(sg, qany_1, qlo_1, qhi_1, c0, BN);
    };
    auto used = [&](int j) { return kind_of(0, j) != TILE_EMPTY || kind_of(1, j) != TILE_EMPTY; };
    auto next_used = [&](int j) {
        ++j;
        while (j < n_kv_tiles && !used(j)) ++j;
        return j;
    };

    // ---- setup
    if (warp == 0 && lane == 0) {
        mbar_init(bar(L::B_Q), 1);
        for (int i = 0; i < L::KST; ++i) {
            mbar_init(bar(L::B_KF + i), 1);
            mbar_init(bar(L::B_KE + i), 1);
        }
        for (int i = 0; i < L::VST; ++i) {
            mbar_init(bar(L::B_VF + i), 1);
            mbar_init(bar(L::B_VE + i), 1);
        }
        for (int t = 0; t < 2; ++t) {
            mbar_init(bar(L::B_S + t), 1);
            mbar_init(bar(L::B_P + t), 128);
            mbar_init(bar(L::B_O + t), 1);
        }
        fence_barrier_init();
        tma_prefetch_desc(&tm_q);
        tma_prefetch_desc(&tm_k);
        tma_prefetch_desc(&tm_v);
    }
    if (warp == 1) {
        tmem_alloc(smem_u32(tmem_slot), 512);
        tmem_relinquish();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp < 4) {
        setmaxnreg_dec88();
        if (warp == 0) {
            // ================= TMA producer =================
            if (elect_one()) {
                const uint64_t pol_kv = policy_evict_last();
                mbar_expect_tx(bar(L::B_Q), 2 * L::TILE);
                for (int b = 0; b < L::NBOX; ++b) {
                    tma_load_3d(sQ + b * kBoxBytes, &tm_q, bar(L::B_Q), b * 64, head_0, static_cast<int>(row0_0));
                    tma_load_3d(sQ + L::TILE + b * kBoxBytes, &tm_q, bar(L::B_Q), b * 64, head_1,
                                static_cast<int>(row0_1));
                }
                int it = 0;
                for (int j = next_used(-1); j < n_kv_tiles; j = next_used(j), ++it) {
                    const int ks = it % L::KST, vs = it % L::VST;
                    mbar_wait(bar(L::B_KE + ks), ((it / L::KST) & 1) ^ 1);
                    mbar_expect_tx(bar(L::B_KF + ks), L::TILE);
                    for (int b = 0; b < L::NBOX; ++b)
                        tma_load_3d_hint(sK + ks * L::TILE + b * kBoxBytes, &tm_k, bar(L::B_KF + ks), b * 64,
                                         kvh, j * BN, pol_kv);
                    mbar_wait(bar(L::B_VE + vs), ((it / L::VST) & 1) ^ 1);
                    mbar_expect_tx(bar(L::B_VF + vs), L::TILE);
                    for (int b = 0; b < L::NBOX; ++b)
                        tma_load_3d_hint(sV + vs * L::TILE + b * kBoxBytes, &tm_v, bar(L::B_VF + vs), b * 64,
                                         kvh, j * BN, pol_kv);
                }
            }
            __syncwarp();
        } else if (warp == 1) {
            // ================= MMA issuer (one thread) =================
            if (elect_one()) {
                constexpr uint32_t idesc_qk = idesc_bf16_f32(BM, BN, false, false);
                constexpr uint32_t idesc_pv = idesc_bf16_f32(BM, HD, false, true);
                auto issue_qk = [&](int t, int ks) {
#pragma unroll
                    for (int kk = 0; kk < HD / 16; ++kk) {
                        const uint32_t off = (kk / 4) * kBoxBytes + (kk % 4) * 32;
                        const uint64_t a = umma_desc_sw128(sQ + t * L::TILE + off, 16, 1024);
                        const uint64_t b = umma_desc_sw128(sK + ks * L::TILE + off, 16, 1024);
                        mma_ss(tmem + (t ? COL_S1 : COL_S0), a, b, idesc_qk, kk > 0);
                    }
                };
                auto issue_pv = [&](int t, int vs, bool acc) {
#pragma unroll
                    for (int kk = 0; kk < BN / 16; ++kk) {
                        // V tile: [128 kv rows][64 d] per box, MN-major B operand; K step = 16 rows
                        const uint64_t b = umma_desc_sw128(sV + vs * L::TILE + kk * 16 * 128, kBoxBytes, 1024);
                        mma_ts(tmem + (t ? COL_O1 : COL_O0), tmem + (t ? COL_S1 : COL_S0) + kk * 8, b, idesc_pv,
                               (acc || kk > 0) ? 1u : 0u);
                    }
                };
                mbar_wait(bar(L::B_Q), 0);
                tc_fence_after();
                int j = next_used(-1);
                int it = 0;
                if (j < n_kv_tiles) {
                    mbar_wait(bar(L::B_KF + 0), 0);
                    tc_fence_after();
                    issue_qk(0, 0);
                    mma_commit(bar(L::B_S + 0));
                    issue_qk(1, 0);
                    mma_commit(bar(L::B_S + 1));
                    mma_commit(bar(L::B_KE + 0));
                }
                while (j < n_kv_tiles) {
                    const int jn = next_used(j);
                    const int vs = it % L::VST;
                    const int ks_n = (it + 1) % L::KST;
                    mbar_wait(bar(L::B_VF + vs), (it / L::VST) & 1);
                    mbar_wait(bar(L::B_P + 0), it & 1);
                    tc_fence_after();
                    issue_pv(0, vs, it > 0);
                    if (jn < n_kv_tiles) {
                        mbar_wait(bar(L::B_KF + ks_n), ((it + 1) / L::KST) & 1);
                        tc_fence_after();
                        issue_qk(0, ks_n);
                        mma_commit(bar(L::B_S + 0));
                    } else {
                        mma_commit(bar(L::B_O + 0));
                    }
                    mbar_wait(bar(L::B_P + 1), it & 1);
                    tc_fence_after();
                    issue_pv(1, vs, it > 0);
                    mma_commit(bar(L::B_VE + vs));
                    if (jn < n_kv_tiles) {
                        issue_qk(1, ks_n);
                        mma_commit(bar(L::B_S + 1));
                        mma_commit(bar(L::B_KE + ks_n));
                    } else {
                        mma_commit(bar(L::B_O + 1));
                    }
                    j = jn;
                    ++it;
                }
            }
            __syncwarp();
        }
    } else {
        // ================= softmax + epilogue, one warpgroup per query tile =================
        setmaxnreg_inc208();
        const int t = (warp >> 2) - 1;
        const int quad = warp & 3;
        const int r = quad * 32 + lane;
        const int64_t row = (t ? row0_1 : row0_0) + r;
        const bool row_ok = row < sg.nq;
        const int64_t my_qpos = row_ok ? seg_qpos(sg, row) : INT64_MAX;
        const uint32_t lane_off = static_cast<uint32_t>(quad * 32) << 16;
        const uint32_t tS = tmem + lane_off + (t == 0 ? COL_S0 : COL_S1);
        const uint32_t tO = tmem + lane_off + (t == 0 ? COL_O0 : COL_O1);
        const float sl2 = p.scale_log2;
        float m = -INFINITY, l = 0.f;
        int it = 0;
        for (int j = next_used(-1); j < n_kv_tiles; j = next_used(j), ++it) {
            const int kind = kind_of(t, j);
            mbar_wait(bar(L::B_S + t), it & 1);
            tc_fence_after();
            if (kind == TILE_EMPTY) {
                uint32_t z[16];
#pragma unroll
                for (int i = 0; i < 16; ++i) z[i] = 0u;
#pragma unroll
                for (int ch = 0; ch < 4; ++ch) tmem_st16(tS + ch * 16, z);
            } else {
                uint32_t s[4][32];
#pragma unroll
                for (int ch = 0; ch < 4; ++ch) tmem_ld32(tS + ch * 32, s[ch]);
                tc_wait_ld();
                if (kind == TILE_PARTIAL) {
                    const int64_t c0 = static_cast<int64_t>(j) * BN;
#pragma unroll
                    for (int ch = 0; ch < 4; ++ch)
#pragma unroll
                        for (int i = 0; i < 32; ++i)
                            if (!seg_visible(sg, c0 + ch * 32 + i, my_qpos)) s[ch][i] = __float_as_uint(-INFINITY);
                }
                float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
                for (int ch = 0; ch < 4; ++ch)
#pragma unroll
                    for (int i = 0; i < 32; i += 2) {
                        mx0 = fmaxf(mx0, __uint_as_float(s[ch][i]));
                        mx1 = fmaxf(mx1, __uint_as_float(s[ch][i + 1]));
                    }
                const float m_new = fmaxf(m, fmaxf(mx0, mx1) * sl2);
                const bool need = m_new > m + 8.0f;
                if (__any_sync(0xFFFFFFFFu, need)) {
                    const float alpha = need ? ex2(m - m_new) : 1.0f;
                    if (need) {
                        l *= alpha;
                        m = m_new;
                    }
                    if (it > 0) {
#pragma unroll
                        for (int c = 0; c < HD / 32; ++c) {
                            uint32_t o[32];
                            tmem_ld32(tO + c * 32, o);
                            tc_wait_ld();
#pragma unroll
                            for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
                            tmem_st32(tO + c * 32, o);
                        }
                    }
                }
                const float m_use = (m == -INFINITY) ? 0.f : m;
                float l0 = 0.f, l1 = 0.f;
#pragma unroll
                for (int ch = 0; ch < 4; ++ch) {
                    uint32_t pk[16];
#pragma unroll
                    for (int i = 0; i < 16; ++i) {
                        const float p0 = ex2(fmaf(__uint_as_float(s[ch][2 * i]), sl2, -m_use));
                        const float p1 = ex2(fmaf(__uint_as_float(s[ch][2 * i + 1]), sl2, -m_use));
                        l0 += p0;
                        l1 += p1;
                        pk[i] = pack_bf16(p0, p1);
                    }
                    tmem_st16(tS + ch * 16, pk);
                }
                l += l0 + l1;
            }
            tc_wait_st();
            tc_fence_before();
            mbar_arrive(bar(L::B_P + t));
        }

        // ---------------- epilogue: normalise, then write / LSE-merge (R3) ----------------
        const int n_used = it;
        if (n_used > 0) {
            mbar_wait(bar(L::B_O + t), 0);
            tc_fence_after();
        }
        const int h = t ? head_1 : head_0;
        const float inv_l = l > 0.f ? 1.0f / l : 0.f;
        const float lse_b = l > 0.f ? (m + __log2f(l)) * 0.69314718055994530942f : -INFINITY;
        const int64_t nq = sg.nq;
        const size_t orow = (static_cast<size_t>(row_ok ? row : 0) * p.Hq + h) * HD;
        float wa = 0.f, wb = 1.f, lse_out = lse_b;
        if (p.mode == CDSP_ATTN_MID || p.mode == CDSP_ATTN_LAST) {
            const float lse_a = row_ok ? p.lse_acc[static_cast<size_t>(h) * nq + row] : -INFINITY;
            merge_weights(lse_a, lse_b, wa, wb, lse_out);
        }
        const float sb = wb * inv_l;
#pragma unroll 1
        for (int c = 0; c < HD / 32; ++c) {
            uint32_t o[32];
            if (n_used > 0) {
                tmem_ld32(tO + c * 32, o);
                tc_wait_ld();
            } else {
#pragma unroll
                for (int i = 0; i < 32; ++i) o[i] = 0u;
            }
            if (!row_ok) continue;
            float v[32];
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(o[i]) * sb;
            if (p.mode == CDSP_ATTN_MID || p.mode == CDSP_ATTN_LAST) {
                const float4* a4 = reinterpret_cast<const float4*>(p.o_acc + orow + c * 32);
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    const float4 a = a4[i];
                    v[4 * i + 0] = fmaf(wa, a.x, v[4 * i + 0]);
                    v[4 * i + 1] = fmaf(wa, a.y, v[4 * i + 1]);
                    v[4 * i + 2] = fmaf(wa, a.z, v[4 * i + 2]);
                    v[4 * i + 3] = fmaf(wa, a.w, v[4 * i + 3]);
                }
            }
            if (p.mode == CDSP_ATTN_FIRST || p.mode == CDSP_ATTN_MID) {
                float4* d4 = reinterpret_cast<float4*>(p.o_acc + orow + c * 32);
#pragma unroll
                for (int i = 0; i < 8; ++i) d4[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
            } else {
                uint4* d4 = reinterpret_cast<uint4*>(p.out + orow + c * 32);
#pragma unroll
                for (int i = 0; i < 4; ++i)
                    d4[i] = make_uint4(pack_bf16(v[8 * i + 0], v[8 * i + 1]), pack_bf16(v[8 * i + 2], v[8 * i + 3]),
                                       pack_bf16(v[8 * i + 4], v[8 * i + 5]), pack_bf16(v[8 * i + 6], v[8 * i + 7]));
            }
        }
        if (row_ok) {
            const size_t li = static_cast<size_t>(h) * nq + row;
            if (p.mode == CDSP_ATTN_FIRST || p.mode == CDSP_ATTN_MID) {
                p.lse_acc[li] = lse_out;
            } else if (p.lse) {
                p.lse[li] = lse_out;
            }
        }
    }

    // ---- teardown
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

// ------------------------------------------------------------------ host side
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn get_encode_fn() {
    static EncodeTiledFn fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(p);
    }
    return fn;
}

// [T, H, D] bf16 tensor, box = 128 rows x 1 head x 64 d, 128-byte swizzle.
cdsp_status make_map(CUtensorMap* m, const void* base, int64_t T, int H, int D) {
    EncodeTiledFn enc = get_encode_fn();
    CDSP_REQUIRE(enc != nullptr, CDSP_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    CDSP_REQUIRE((reinterpret_cast<uintptr_t>(base) & 15u) == 0, CDSP_ERR_INVALID,
                 "TMA base pointer must be 16-byte aligned");
    cuuint64_t dims[3] = {static_cast<cuuint64_t>(D), static_cast<cuuint64_t>(H),
                          static_cast<cuuint64_t>(T > 0 ? T : 1)};
    cuuint64_t strides[2] = {static_cast<cuuint64_t>(D) * 2, static_cast<cuuint64_t>(H) * D * 2};
    cuuint32_t box[3] = {64, 1, 128};
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    CDSP_REQUIRE(r == CUDA_SUCCESS, CDSP_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", static_cast<int>(r));
    return CDSP_OK;
}

template <int HD>
cdsp_status launch_tc(const AttnArgs& a, cudaStream_t st) {
    using Lt = Layout<HD>;
    static bool attr_set = false;
    if (!attr_set) {
        CDSP_CUDA(cudaFuncSetAttribute(attn_tc_kernel<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, Lt::SMEM));
        attr_set = true;
    }
    CUtensorMap mq, mk, mv;
    CDSP_CHECK_STATUS(make_map(&mq, a.q, a.seg.nq, a.Hq, HD));
    const void* kb = a.seg.nkv > 0 ? a.k : a.q;  // nkv == 0: map never dereferenced
    const void* vb = a.seg.nkv > 0 ? a.v : a.q;
    CDSP_CHECK_STATUS(make_map(&mk, kb, a.seg.nkv, a.seg.nkv > 0 ? a.Hkv : a.Hq, HD));
    CDSP_CHECK_STATUS(make_map(&mv, vb, a.seg.nkv, a.seg.nkv > 0 ? a.Hkv : a.Hq, HD));
    TcParams p;
    p.seg = a.seg;
    p.Hq = a.Hq;
    p.Hkv = a.Hkv;
    p.g = a.Hq / a.Hkv;
    p.pair_heads = (p.g % 2 == 0) ? 1 : 0;
    p.n_hg = p.pair_heads ? a.Hq / 2 : a.Hq;
    const int64_t rows_per_cta = p.pair_heads ? BM : 2 * BM;
    p.n_rb = static_cast<int>((a.seg.nq + rows_per_cta - 1) / rows_per_cta);
    p.scale_log2 = a.scale * 1.4426950408889634f;
    p.mode = a.mode;
    p.o_acc = a.o_acc;
    p.lse_acc = a.lse_acc;
    p.out = static_cast<__nv_bfloat16*>(a.out);
    p.lse = a.lse;
    const int64_t grid = static_cast<int64_t>(p.n_rb) * p.n_hg;
    if (grid == 0) return CDSP_OK;
    CDSP_REQUIRE(grid < (1ll << 31), CDSP_ERR_SHAPE, "grid too large");
    attn_tc_kernel<HD><<<static_cast<unsigned>(grid), kThreads, Lt::SMEM, st>>>(mq, mk, mv, p);
    CDSP_CUDA(cudaGetLastError());
    return CDSP_OK;
}

}  // namespace

cdsp_status launch_attention_tc(const AttnArgs& a, cudaStream_t st) {
    if (a.D == 128) return launch_tc<128>(a, st);
    if (a.D == 64) return launch_tc<64>(a, st);
    CDSP_FAIL(CDSP_ERR_SHAPE, "head dim %d not supported (64 or 128)", a.D);
}

}  // namespace cdsp
