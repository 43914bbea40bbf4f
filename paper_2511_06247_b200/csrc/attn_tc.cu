// attn_tc.cu — K*1: bf16 block attention for one ring step on sm_100a tensor cores.
//
// Computes, for a query shard and one KV block (history + a current-chunk shard), exact
// softmax attention under the position mask of attn_common.cuh, and writes or LSE-merges
// the result (cdsp_attn_mode).  This is the per-step compute of ring attention
// (§2.3: each instance "interact[s] local query tensors with full key-value
// tensors"), extended to historical tokens as Tetris does (§6: "we extend Flash
// Attention [7] to support zigzag ring attention for historical tokens").
//
// B200 design (not the paper's A100 FlashAttention-2), from measurements on the box:
//  * tcgen05.mma M=128 reaches the full 8192 FLOP/clk/SM only for N >= 128 (N=64: ~48 clk
//    per K=16 step instead of 32; tools/mma_rate.cu), so S = Q K^T uses 128-key tiles.
//  * MUFU.EX2 issues 16 lanes/clk/SM (tools/exp_rate.cu): the 16384 exponentials of a
//    128x128 tile take 1024 clk, exactly the two MMAs of that tile.  3/8 of them therefore
//    run as a cubic on the FMA pipe, and the softmax must spend almost no issue slots on
//    anything else.  One thread owns one query row (all 128 columns of S in registers):
//    the row max needs no cross-warp exchange and per-tile bookkeeping (waits, arrives,
//    TMEM addressing) is paid by 4 warps per tile instead of 16.
//  * one CTA = two 128-row query tiles (Q0, Q1) of one head, 11 warps:
//      warps 0-3   softmax + epilogue of Q0 (warp w owns TMEM lanes 32*(w%4)..)
//      warps 4-7   softmax + epilogue of Q1
//      warp 8      TMA producer: Q0, Q1 once, then K tiles (2 stages)
//      warp 9      TMA producer: V tiles (2 stages)
//      warp 10     TMEM allocator + tcgen05.mma issuer (warp-uniform loop, one lane issues)
//    The tensor pipe alternates [O0 += P0 V_{j-1}, S0 = Q0 K_j^T] and [O1 += P1 V_{j-1},
//    S1 = Q1 K_j^T]: while it works for one query tile the other tile's softmax runs, so
//    each softmax group has a full half-period (two MMAs) for its 128x128 tile.
//  * TMEM (512 cols): O0 [0,128), O1 [128,256), S0 [256,384), S1 [384,512).  P (bf16) is
//    written over its own S columns and is the A operand of PV straight from TMEM; the
//    next S into those columns is issued after that PV on the same in-order tensor pipe.
//    S_t(j) is committed after PV_t(j-1), so when the softmax sees S_t(j), O_t is stable.
//  * lazy rescaling: the running max only moves when it grows by > 8 (log2 units); O is
//    rescaled in TMEM after P is stored (registers of S are dead by then).
//  * masks from segment descriptors: empty tiles are skipped per query tile, full tiles run
//    mask-free, diagonal / ragged tiles build per-row 32-bit column masks from the three
//    visible intervals (history, segment 0, segment 1).
#include <cuda.h>
#include <cuda_bf16.h>

#include <climits>
#include <cstdio>
#include <cstdlib>

#include "attn_common.cuh"
#include "common.cuh"
#include "internal.h"
#include "ptx.cuh"

#ifndef CDSP_EMU_MASK
#define CDSP_EMU_MASK 0x52
#endif

namespace cdsp {
using namespace ptx;

namespace {

constexpr int kThreads = 352;           // 11 warps
constexpr int BQ = 128;                 // rows per query tile (TMEM lanes)
constexpr int NQT = 2;                  // query tiles per CTA
constexpr int BM = BQ * NQT;            // query rows per CTA
constexpr int BN = 128;                 // KV rows per tile
constexpr int kBox = 128 * 128;         // TMA box: 128 rows x 64 bf16 (128-byte swizzle rows)
constexpr int kSchedMax = 8192;         // KV tiles per launch (1M keys)
constexpr int W_K = 8, W_V = 9, W_MMA = 10;
constexpr int kSchedWarps = 8;          // warps 0-7 classify the KV tiles at setup

template <int HD>
struct Layout {
    static constexpr int NBOX = HD / 64;
    static constexpr int TILE = kBox * NBOX;  // one 128-row tile of Q, K or V
    static constexpr int KST = 2, VST = 2;
    static constexpr int OFF_Q = 0;
    static constexpr int OFF_K = OFF_Q + NQT * TILE;
    static constexpr int OFF_V = OFF_K + KST * TILE;
    static constexpr int OFF_BAR = OFF_V + VST * TILE;
    // q_full[2], k_full[KST], k_empty[KST], v_full[VST], v_empty[VST], s_full[2], p_full[2], o_full[2]
    static constexpr int B_Q = 0, B_KF = B_Q + NQT, B_KE = B_KF + KST, B_VF = B_KE + KST, B_VE = B_VF + VST,
                         B_SF = B_VE + VST, B_PF = B_SF + NQT, B_OF = B_PF + NQT, NBAR = B_OF + NQT;
    static constexpr int OFF_TMEM_SLOT = OFF_BAR + NBAR * 8;
    static constexpr int OFF_JR = OFF_TMEM_SLOT + 16;   // used-tile range per setup warp: (min, max+1)
    static constexpr int OFF_SCHED = OFF_JR + 8 * kSchedWarps;
    static constexpr int SMEM = OFF_SCHED + kSchedMax + 1024;  // + alignment slack
};

__host__ __device__ constexpr uint32_t col_o(int t) { return 128u * t; }
__host__ __device__ constexpr uint32_t col_s(int t) { return 256u + 128u * t; }

struct TcParams {
    cdsp_segments seg;
    int Hq, Hkv, g, n_rb;
    float scale_log2;
    int mode;
    float* o_acc;
    float* lse_acc;
    __nv_bfloat16* out;
    float* lse;
};

// Debug timeline (build with -DCDSP_KTRACE): per-CTA phase stamps (globaltimer) and SM id,
// dumped by the host when CDSP_TRACE=<file> is set.
#ifdef CDSP_KTRACE
__device__ unsigned long long g_cta[65536 * 8];  // start, end, smid, used tiles, setup, 1st S, loop end, epi end
__device__ __forceinline__ unsigned long long gtime_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ unsigned long long g_it[4 * 512 * 16];  // CTAs 0..3, first 512 iterations, 16 slots
#define KTRACE(slot, iter)                                                                             \
    do {                                                                                               \
        if (blockIdx.x < 4 && (iter) < 512)                                                            \
            g_it[(static_cast<size_t>(blockIdx.x) * 512 + (iter)) * 16 + (slot)] = clock64();          \
    } while (0)
#define CTA_STAMP(slot)                                                                           \
    do {                                                                                          \
        if (blockIdx.x < 65536) g_cta[static_cast<size_t>(blockIdx.x) * 8 + (slot)] = gtime_ns(); \
    } while (0)
#else
#define KTRACE(slot, iter) \
    do {                   \
    } while (0)
#define CTA_STAMP(slot) \
    do {                \
    } while (0)
#endif

// ---- packed fp32x2 arithmetic (FFMA2 / FADD2 on sm_100)
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
    float2 d;
    asm("{\n\t.reg .b64 ra, rb, rc, rd;\n\t"
        "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\tmov.b64 rc, {%6, %7};\n\t"
        "fma.rn.f32x2 rd, ra, rb, rc;\n\tmov.b64 {%0, %1}, rd;\n\t}"
        : "=f"(d.x), "=f"(d.y)
        : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
    return d;
}
__device__ __forceinline__ float2 fadd2(float2 a, float2 b) {
    float2 d;
    asm("{\n\t.reg .b64 ra, rb, rd;\n\t"
        "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
        "add.f32x2 rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;\n\t}"
        : "=f"(d.x), "=f"(d.y)
        : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
    return d;
}

// 2^x for a pair on the FMA pipe: n = rint(x) by the 1.5*2^23 magic (which also leaves n in
// the low mantissa bits of t), f = x - n in [-1/2, 1/2], 2^f by a cubic fitted for minimax
// relative error on [-1/2, 1/2] (7.5e-5), 2^n added to the exponent field.
__device__ __forceinline__ float2 ex2_fma2(float2 x) {
    x.x = fmaxf(x.x, -126.0f);
    x.y = fmaxf(x.y, -126.0f);
    const float2 t = fadd2(x, make_float2(12582912.0f, 12582912.0f));
    const float2 n = fadd2(t, make_float2(-12582912.0f, -12582912.0f));
    const float2 f = fadd2(x, make_float2(-n.x, -n.y));
    float2 q = ffma2(make_float2(0.05517138913273811f, 0.05517138913273811f), f,
                     make_float2(0.24261070787906647f, 0.24261070787906647f));
    q = ffma2(q, f, make_float2(0.6932609677314758f, 0.6932609677314758f));
    q = ffma2(q, f, make_float2(0.9999281167984009f, 0.9999281167984009f));
    return make_float2(__int_as_float(__float_as_int(q.x) + (__float_as_int(t.x) << 23)),
                       __int_as_float(__float_as_int(q.y) + (__float_as_int(t.y) << 23)));
}

// Registers loaded by tcgen05.ld are only valid after tcgen05.wait::ld; tying them to an
// (empty) volatile asm after the wait keeps their uses below it.
__device__ __forceinline__ void reg_tie32(uint32_t* r) {
    asm volatile(""
                 : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]),
                   "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]), "+r"(r[14]),
                   "+r"(r[15]), "+r"(r[16]), "+r"(r[17]), "+r"(r[18]), "+r"(r[19]), "+r"(r[20]), "+r"(r[21]),
                   "+r"(r[22]), "+r"(r[23]), "+r"(r[24]), "+r"(r[25]), "+r"(r[26]), "+r"(r[27]), "+r"(r[28]),
                   "+r"(r[29]), "+r"(r[30]), "+r"(r[31]));
}
__device__ __forceinline__ void tmem_ld32p(uint32_t taddr, uint32_t* r) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
          "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
          "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
          "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
}

__device__ __forceinline__ int clamp_bn(int64_t x) { return x < 0 ? 0 : (x > BN ? BN : static_cast<int>(x)); }
// bits [lo, hi) of the 32 columns starting at `base`
__device__ __forceinline__ uint32_t range_bits(int lo, int hi, int base) {
    const int l = max(lo - base, 0), h = min(hi - base, 32);
    if (l >= h) return 0u;
    const uint32_t hm = h >= 32 ? 0xFFFFFFFFu : ((1u << h) - 1u);
    return hm & ~((1u << l) - 1u);
}

// Mask a partial tile: the KV rows of tile j visible to a query at position qpos are the
// union of [0, b0) (history), [a1, b1) (segment 0 rows with pos <= qpos) and [a2, b2)
// (segment 1 rows with pos <= qpos), tile-relative — seg_visible() written as intervals.
__device__ __forceinline__ void mask_tile(uint32_t* s, const cdsp_segments& sg, int j, int64_t qpos) {
    const int64_t c0 = static_cast<int64_t>(j) * BN;
    const int nk = clamp_bn(sg.nkv - c0);
    const int h = clamp_bn(sg.kv_hist - c0);
    const int64_t e0abs = sg.kv_hist + sg.kv_len0;
    const int e0 = clamp_bn(e0abs - c0);
    const int lim0 = clamp_bn(qpos - sg.kv_pos0 + sg.kv_hist + 1 - c0);
    const int lim1 = clamp_bn(qpos - sg.kv_pos1 + e0abs + 1 - c0);
    const int b0 = min(h, nk);
    const int a1 = h, b1 = min(min(e0, lim0), nk);
    const int a2 = e0, b2 = min(nk, lim1);
#pragma unroll
    for (int w = 0; w < BN / 32; ++w) {
        const uint32_t mk = range_bits(0, b0, 32 * w) | range_bits(a1, b1, 32 * w) | range_bits(a2, b2, 32 * w);
#pragma unroll
        for (int i = 0; i < 32; ++i)
            if (!((mk >> i) & 1u)) s[32 * w + i] = __float_as_uint(-INFINITY);
    }
}

template <int HD>
__global__ void __maxnreg__(168)
    attn_tc_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                   const __grid_constant__ CUtensorMap tm_v, const TcParams p) {
    using L = Layout<HD>;
    extern __shared__ uint8_t smem_raw[];
#ifdef CDSP_KTRACE
    const unsigned long long t_start = gtime_ns();
#endif
    // 1024-byte alignment for the 128B-swizzle atoms
    const uint32_t raw_addr = smem_u32(smem_raw);
    uint8_t* smem = smem_raw + ((1024u - (raw_addr & 1023u)) & 1023u);
    const uint32_t sbase = smem_u32(smem);
    const uint32_t sQ = sbase + L::OFF_Q, sK = sbase + L::OFF_K, sV = sbase + L::OFF_V;
    const uint32_t bar0 = sbase + L::OFF_BAR;
    auto bar = [&](int i) { return bar0 + 8u * static_cast<uint32_t>(i); };
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + L::OFF_TMEM_SLOT);
    uint8_t* sched = smem + L::OFF_SCHED;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const cdsp_segments& sg = p.seg;

    // ---- work unit: head-major (the ~148 CTAs in flight share one head's K/V, which stays
    // L2-resident), heavy row blocks first within a head (causal work grows with the row)
    const int head = static_cast<int>(blockIdx.x) / p.n_rb;
    const int rb = p.n_rb - 1 - static_cast<int>(blockIdx.x) % p.n_rb;
    const int kvh = head / p.g;
    const int64_t row0 = static_cast<int64_t>(rb) * BM;
    const int n_kv_tiles = static_cast<int>((sg.nkv + BN - 1) / BN);
    const bool q1_rows = row0 + BQ < sg.nq;

    // ---- setup
    if (warp == W_K) {
        if (lane == 0) {
            for (int t = 0; t < NQT; ++t) mbar_init(bar(L::B_Q + t), 1);
            for (int i = 0; i < L::KST; ++i) {
                mbar_init(bar(L::B_KF + i), 1);
                mbar_init(bar(L::B_KE + i), 1);
            }
            for (int i = 0; i < L::VST; ++i) {
                mbar_init(bar(L::B_VF + i), 1);
                mbar_init(bar(L::B_VE + i), 1);
            }
            for (int t = 0; t < NQT; ++t) {
                mbar_init(bar(L::B_SF + t), 1);
                mbar_init(bar(L::B_PF + t), 4);
                mbar_init(bar(L::B_OF + t), 1);
            }
            fence_barrier_init();
            tma_prefetch_desc(&tm_q);
            tma_prefetch_desc(&tm_k);
            tma_prefetch_desc(&tm_v);
            // Q does not depend on the schedule: start its loads now
            for (int t = 0; t < (q1_rows ? 2 : 1); ++t) {
                mbar_expect_tx(bar(L::B_Q + t), L::TILE);
                for (int b = 0; b < L::NBOX; ++b)
                    tma_load_3d(sQ + t * L::TILE + b * kBox, &tm_q, bar(L::B_Q + t), b * 64, head,
                                static_cast<int>(row0 + t * BQ));
            }
        }
    } else if (warp == W_MMA) {
        tmem_alloc(smem_u32(tmem_slot), 512);
        tmem_relinquish();
    } else if (warp < kSchedWarps) {
        // KV-tile schedule: sched[j] = kind for Q0 | kind for Q1 << 2 (0 = skip)
        int64_t qlo0, qhi0, qlo1, qhi1;
        bool qany0, qany1;
        seg_qrange(sg, row0, row0 + BQ, qlo0, qhi0, qany0);
        seg_qrange(sg, row0 + BQ, row0 + BM, qlo1, qhi1, qany1);
        int jmin = INT_MAX, jmax = 0;
        for (int j = warp * 32 + lane; j < n_kv_tiles; j += kSchedWarps * 32) {
            const int64_t c0 = static_cast<int64_t>(j) * BN;
            const int k = seg_tile_kind(sg, qany0, qlo0, qhi0, c0, BN) | (seg_tile_kind(sg, qany1, qlo1, qhi1, c0, BN) << 2);
            sched[j] = static_cast<uint8_t>(k);
            if (k != 0) {
                jmin = min(jmin, j);
                jmax = max(jmax, j + 1);
            }
        }
        for (int o = 16; o > 0; o >>= 1) {
            jmin = min(jmin, __shfl_xor_sync(0xFFFFFFFFu, jmin, o));
            jmax = max(jmax, __shfl_xor_sync(0xFFFFFFFFu, jmax, o));
        }
        if (lane == 0) {
            reinterpret_cast<int*>(smem + L::OFF_JR)[2 * warp] = jmin;
            reinterpret_cast<int*>(smem + L::OFF_JR)[2 * warp + 1] = jmax;
        }
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    // the used KV tiles lie in [j_lo, j_hi) (sched[j] == 0 marks skipped tiles inside it)
    int j_lo = INT_MAX, j_hi = 0;
    {
        const int* jr = reinterpret_cast<const int*>(smem + L::OFF_JR);
#pragma unroll
        for (int w = 0; w < kSchedWarps; ++w) {
            j_lo = min(j_lo, jr[2 * w]);
            j_hi = max(j_hi, jr[2 * w + 1]);
        }
    }
    if (threadIdx.x == 0) CTA_STAMP(4);

    if (warp == W_K || warp == W_V) {
        // ======== TMA producers: K and V in independent rings (a K load never waits behind a
        // V stage); one lane issues, the warp runs the loop ========
        const bool is_k = warp == W_K;
        const int nst = is_k ? L::KST : L::VST;
        const uint32_t s0 = is_k ? sK : sV;
        const int bfull = is_k ? L::B_KF : L::B_VF, bempty = is_k ? L::B_KE : L::B_VE;
        const void* map = is_k ? static_cast<const void*>(&tm_k) : static_cast<const void*>(&tm_v);
        const uint64_t pol_kv = policy_evict_last();
        int it = 0;
        for (int j = j_lo; j < j_hi; ++j) {
            if (sched[j] == 0) continue;
            const int st = it % nst;
            mbar_wait(bar(bempty + st), ((it / nst) & 1) ^ 1);
            if (elect_one()) {
                mbar_expect_tx(bar(bfull + st), L::TILE);
                for (int b = 0; b < L::NBOX; ++b)
                    tma_load_3d_hint(s0 + st * L::TILE + b * kBox, map, bar(bfull + st), b * 64, kvh, j * BN, pol_kv);
            }
            __syncwarp();
            ++it;
        }
    } else if (warp == W_MMA) {
        // ================= MMA issuer (warp-uniform loop, one lane issues) =================
        constexpr uint32_t idesc_qk = idesc_bf16_f32(BQ, BN, false, false);
        constexpr uint32_t idesc_pv = idesc_bf16_f32(BQ, HD, false, true);
        const uint64_t dq0 = umma_desc_sw128(sQ, 16, 1024);
        const uint64_t dk0 = umma_desc_sw128(sK, 16, 1024);
        const uint64_t dv0 = umma_desc_sw128(sV, kBox, 1024);
        // S_t = Q_t K^T: M=128, N=128, K=HD in steps of 16 (32 B inside a 128-B swizzle row)
        auto issue_qk = [&](int t, int ks) {
            const uint64_t dk = dk0 + static_cast<uint64_t>((ks * L::TILE) >> 4);
            const uint64_t dq = dq0 + static_cast<uint64_t>((t * L::TILE) >> 4);
#pragma unroll
            for (int kk = 0; kk < HD / 16; ++kk) {
                const uint64_t off = static_cast<uint64_t>(((kk / 4) * kBox + (kk % 4) * 32) >> 4);
                mma_ss(tmem + col_s(t), dq + off, dk + off, idesc_qk, kk > 0 ? 1u : 0u);
            }
        };
        // O_t += P_t V: M=128, N=HD, K=128 keys in steps of 16 (V rows, 2048 B); P_t is bf16
        // in the S_t columns (8 TMEM columns per 16 keys)
        auto issue_pv = [&](int t, int vs, bool acc) {
            const uint64_t dv = dv0 + static_cast<uint64_t>((vs * L::TILE) >> 4);
#pragma unroll
            for (int kk = 0; kk < BN / 16; ++kk)
                mma_ts(tmem + col_o(t), tmem + col_s(t) + kk * 8, dv + static_cast<uint64_t>((kk * 16 * 128) >> 4),
                       idesc_pv, (acc || kk > 0) ? 1u : 0u);
        };
        // Iteration `it` (union tile j_it): for t = 0, 1: O_t += P_t(j_{it-1}) V_{it-1} (if
        // query tile t used j_{it-1}), then S_t = Q_t K_{it}^T (if it uses j_it).  K stage it
        // is released after its S's, V stage it-1 after its PVs (commit = all prior MMAs).
        int pv0 = 0, pv1 = 0;      // PVs issued per query tile (P_full phases consumed)
        bool q0 = false, q1 = false;
        int prev_kinds = 0, it = 0;
        int j = j_lo;
        while (j < j_hi && sched[j] == 0) ++j;
        for (;;) {
            const bool have = j < j_hi;
            const int kinds = have ? sched[j] : 0;
            const int last_pv_t = (prev_kinds >> 2) ? 1 : 0;
            bool k_waited = false, v_waited = false;
#pragma unroll
            for (int t = 0; t < NQT; ++t) {
                if ((prev_kinds >> (2 * t)) & 3) {
                    int& pv = t == 0 ? pv0 : pv1;
                    mbar_wait(bar(L::B_PF + t), pv & 1);
                    if (!v_waited) {
                        mbar_wait(bar(L::B_VF + (it - 1) % L::VST), ((it - 1) / L::VST) & 1);
                        v_waited = true;
                    }
                    tc_fence_after();
                    if (elect_one()) {
                        KTRACE(8 + 2 * t, it);
                        issue_pv(t, (it - 1) % L::VST, pv > 0);
                        if (t == last_pv_t) mma_commit(bar(L::B_VE + (it - 1) % L::VST));
                    }
                    __syncwarp();
                    ++pv;
                }
                if ((kinds >> (2 * t)) & 3) {
                    bool& qr = t == 0 ? q0 : q1;
                    if (!qr) {
                        mbar_wait(bar(L::B_Q + t), 0);
                        qr = true;
                    }
                    if (!k_waited) {
                        mbar_wait(bar(L::B_KF + it % L::KST), (it / L::KST) & 1);
                        k_waited = true;
                    }
                    tc_fence_after();
                    if (elect_one()) {
                        KTRACE(9 + 2 * t, it);
                        issue_qk(t, it % L::KST);
                        mma_commit(bar(L::B_SF + t));
                    }
                    __syncwarp();
                }
            }
            if (!have) break;
            if (elect_one()) mma_commit(bar(L::B_KE + it % L::KST));
            __syncwarp();
            prev_kinds = kinds;
            ++it;
            ++j;
            while (j < j_hi && sched[j] == 0) ++j;
        }
        if (elect_one()) {
            mma_commit(bar(L::B_OF + 0));
            mma_commit(bar(L::B_OF + 1));
        }
        __syncwarp();
    } else if (warp < 4 * NQT) {
        // ================= softmax + epilogue: thread = one query row of tile t =================
        const int t = warp >> 2;
        const int quad = warp & 3;  // TMEM lane quadrant
        const int r = quad * 32 + lane;
        const int64_t row = row0 + t * BQ + r;
        const bool row_ok = row < sg.nq;
        const int64_t my_qpos = row_ok ? seg_qpos(sg, row) : (INT64_MAX >> 2);
        const uint32_t lane_off = static_cast<uint32_t>(quad * 32) << 16;
        const uint32_t tS = tmem + lane_off + col_s(t);
        const uint32_t tO = tmem + lane_off + col_o(t);
        const float sl2 = p.scale_log2;
        float m = -INFINITY;
        float2 lacc0 = make_float2(0.f, 0.f), lacc1 = make_float2(0.f, 0.f);
        int n = 0;
        for (int j = j_lo; j < j_hi; ++j) {
            const int kind = (sched[j] >> (2 * t)) & 3;
            if (kind == 0) continue;
            uint32_t s[BN];
            mbar_wait(bar(L::B_SF + t), n & 1);
            if (lane == 0 && quad == 0) KTRACE(4 * t + 0, n);
            tc_fence_after();
#pragma unroll
            for (int c = 0; c < BN / 32; ++c) tmem_ld32p(tS + 32 * c, s + 32 * c);
            tc_wait_ld();
#pragma unroll
            for (int c = 0; c < BN / 32; ++c) reg_tie32(s + 32 * c);
            if (threadIdx.x == 0 && n == 0) CTA_STAMP(5);
            if (kind == TILE_PARTIAL) mask_tile(s, sg, j, my_qpos);
            float mx;
            {
                float a0 = -INFINITY, a1 = -INFINITY, a2 = -INFINITY, a3 = -INFINITY;
#pragma unroll
                for (int i = 0; i < BN; i += 8) {
                    a0 = fmaxf(a0, fmaxf(__uint_as_float(s[i + 0]), __uint_as_float(s[i + 1])));
                    a1 = fmaxf(a1, fmaxf(__uint_as_float(s[i + 2]), __uint_as_float(s[i + 3])));
                    a2 = fmaxf(a2, fmaxf(__uint_as_float(s[i + 4]), __uint_as_float(s[i + 5])));
                    a3 = fmaxf(a3, fmaxf(__uint_as_float(s[i + 6]), __uint_as_float(s[i + 7])));
                }
                mx = fmaxf(fmaxf(a0, a1), fmaxf(a2, a3));
            }
            const float m_new = fmaxf(m, mx * sl2);
            const bool need = m_new > m + 8.0f;
            float alpha = 1.0f;
            if (need) {
                alpha = ex2(m - m_new);
                lacc0.x *= alpha;
                lacc0.y *= alpha;
                lacc1.x *= alpha;
                lacc1.y *= alpha;
                m = m_new;
            }
            if (lane == 0 && quad == 0) KTRACE(4 * t + 1, n);
            const float m_use = (m == -INFINITY) ? 0.f : m;
            const float2 sc = make_float2(sl2, sl2), nm = make_float2(-m_use, -m_use);
#pragma unroll
            for (int c = 0; c < BN / 32; ++c) {
                uint32_t pk[16];
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                    const float2 x =
                        ffma2(make_float2(__uint_as_float(s[32 * c + 2 * i]), __uint_as_float(s[32 * c + 2 * i + 1])), sc, nm);
                    float2 pp;
                    if ((CDSP_EMU_MASK >> (i % 8)) & 1) {  // pairs on the FMA pipe (default 3/8)
                        pp = ex2_fma2(x);
                    } else {
                        pp.x = ex2(x.x);
                        pp.y = ex2(x.y);
                    }
                    if (i & 1) lacc1 = fadd2(lacc1, pp);
                    else lacc0 = fadd2(lacc0, pp);
                    pk[i] = pack_bf16(pp.x, pp.y);
                }
                tmem_st16(tS + 16 * c, pk);  // P chunk c over S columns already in registers
            }
            if (lane == 0 && quad == 0) KTRACE(4 * t + 2, n);
            // O_t holds PV_t up to the previous tile (committed before this S_t): rescale it
            if (n > 0 && __any_sync(0xFFFFFFFFu, need)) {
#pragma unroll 1
                for (int c = 0; c < HD / 32; ++c) {
                    uint32_t o[32];
                    tmem_ld32p(tO + 32 * c, o);
                    tc_wait_ld();
                    reg_tie32(o);
#pragma unroll
                    for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
                    tmem_st32(tO + 32 * c, o);
                }
            }
            tc_wait_st();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(bar(L::B_PF + t));
            if (lane == 0 && quad == 0) KTRACE(4 * t + 3, n);
            ++n;
        }

        // ---------------- epilogue: normalise, then write / LSE-merge (R3) ----------------
        if (threadIdx.x == 0) CTA_STAMP(6);
        mbar_wait(bar(L::B_OF + t), 0);
        tc_fence_after();
        const float l = (lacc0.x + lacc0.y) + (lacc1.x + lacc1.y);
        const float inv_l = l > 0.f ? 1.0f / l : 0.f;
        const float lse_b = l > 0.f ? (m + __log2f(l)) * 0.69314718055994530942f : -INFINITY;
        const int64_t nq = sg.nq;
        float wa = 0.f, wb = 1.f, lse_out = lse_b;
        const bool merge = p.mode == CDSP_ATTN_MID || p.mode == CDSP_ATTN_LAST;
        const bool to_acc = p.mode == CDSP_ATTN_FIRST || p.mode == CDSP_ATTN_MID;
        if (merge) {
            const float lse_a = row_ok ? p.lse_acc[static_cast<size_t>(head) * nq + row] : -INFINITY;
            merge_weights(lse_a, lse_b, wa, wb, lse_out);
        }
        const float sbw = wb * inv_l;
        const size_t orow = (static_cast<size_t>(row_ok ? row : 0) * p.Hq + head) * HD;
#pragma unroll 1
        for (int c = 0; c < HD / 32; ++c) {
            uint32_t o[32];
            if (n > 0) {
                tmem_ld32p(tO + 32 * c, o);
                tc_wait_ld();
                reg_tie32(o);
            } else {
#pragma unroll
                for (int i = 0; i < 32; ++i) o[i] = 0u;
            }
            if (row_ok) {
                float v[32];
#pragma unroll
                for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(o[i]) * sbw;
                if (merge) {
                    const float4* a4 = reinterpret_cast<const float4*>(p.o_acc + orow + 32 * c);
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        const float4 a = a4[i];
                        v[4 * i + 0] = fmaf(wa, a.x, v[4 * i + 0]);
                        v[4 * i + 1] = fmaf(wa, a.y, v[4 * i + 1]);
                        v[4 * i + 2] = fmaf(wa, a.z, v[4 * i + 2]);
                        v[4 * i + 3] = fmaf(wa, a.w, v[4 * i + 3]);
                    }
                }
                if (to_acc) {
                    float4* d4 = reinterpret_cast<float4*>(p.o_acc + orow + 32 * c);
#pragma unroll
                    for (int i = 0; i < 8; ++i) d4[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
                } else {
                    uint4* d4 = reinterpret_cast<uint4*>(p.out + orow + 32 * c);
#pragma unroll
                    for (int i = 0; i < 4; ++i)
                        d4[i] = make_uint4(pack_bf16(v[8 * i + 0], v[8 * i + 1]), pack_bf16(v[8 * i + 2], v[8 * i + 3]),
                                           pack_bf16(v[8 * i + 4], v[8 * i + 5]), pack_bf16(v[8 * i + 6], v[8 * i + 7]));
                }
            }
        }
        if (row_ok) {
            const size_t li = static_cast<size_t>(head) * nq + row;
            if (to_acc) {
                p.lse_acc[li] = lse_out;
            } else if (p.lse) {
                p.lse[li] = lse_out;
            }
        }
        if (threadIdx.x == 0) CTA_STAMP(7);
    }

#ifdef CDSP_KTRACE
    if (threadIdx.x == 0 && blockIdx.x < 65536) {
        unsigned smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        int nu = 0;
        for (int j = 0; j < n_kv_tiles; ++j) nu += sched[j] != 0;
        g_cta[blockIdx.x * 8 + 0] = t_start;
        g_cta[blockIdx.x * 8 + 2] = smid;
        g_cta[blockIdx.x * 8 + 3] = nu;
    }
#endif
    // ---- teardown
    tc_fence_before();
    __syncthreads();
    if (warp == W_MMA) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
    if (threadIdx.x == 0) CTA_STAMP(1);
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
    CDSP_REQUIRE((a.seg.nkv + BN - 1) / BN <= kSchedMax, CDSP_ERR_CAPACITY, "KV block of %lld rows exceeds %d",
                 static_cast<long long>(a.seg.nkv), kSchedMax * BN);
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
    p.n_rb = static_cast<int>((a.seg.nq + BM - 1) / BM);
    p.scale_log2 = a.scale * 1.4426950408889634f;
    p.mode = a.mode;
    p.o_acc = a.o_acc;
    p.lse_acc = a.lse_acc;
    p.out = static_cast<__nv_bfloat16*>(a.out);
    p.lse = a.lse;
    const int64_t grid = static_cast<int64_t>(p.n_rb) * a.Hq;
    if (grid == 0) return CDSP_OK;
    CDSP_REQUIRE(grid < (1ll << 31), CDSP_ERR_SHAPE, "grid too large");
    attn_tc_kernel<HD><<<static_cast<unsigned>(grid), kThreads, Lt::SMEM, st>>>(mq, mk, mv, p);
    CDSP_CUDA(cudaGetLastError());
#ifdef CDSP_KTRACE
    if (const char* path = getenv("CDSP_TRACE")) {  // debug builds only: synchronous dump
        static unsigned long long c[65536 * 8], it[4 * 512 * 16];
        CDSP_CUDA(cudaStreamSynchronize(st));
        CDSP_CUDA(cudaMemcpyFromSymbol(c, g_cta, sizeof(c)));
        CDSP_CUDA(cudaMemcpyFromSymbol(it, g_it, sizeof(it)));
        if (FILE* f = fopen(path, "wb")) {
            fwrite(c, 1, sizeof(c), f);
            fwrite(it, 1, sizeof(it), f);
            fclose(f);
        }
    }
#endif
    return CDSP_OK;
}

}  // namespace

cdsp_status launch_attention_tc(const AttnArgs& a, cudaStream_t st) {
    if (a.D == 128) return launch_tc<128>(a, st);
    if (a.D == 64) return launch_tc<64>(a, st);
    CDSP_FAIL(CDSP_ERR_SHAPE, "head dim %d not supported (64 or 128)", a.D);
}

}  // namespace cdsp
