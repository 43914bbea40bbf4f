// attn_tc.cu — K*1: bf16 block attention for one ring step on sm_100a tensor cores.
//
// Computes, for a query shard and one KV block (history + a current-chunk shard), exact
// softmax attention under the position mask of attn_common.cuh, and writes or LSE-merges
// the result (cdsp_attn_mode).  This is the per-step compute of ring attention
// (§2.3: each instance "interact[s] local query tensors with full key-value
// tensors"), extended to historical tokens as Tetris does (§6: "we extend Flash
// Attention [7] to support zigzag ring attention for historical tokens").
//
// B200 design (not the paper's A100 FlashAttention-2), measured on the box:
//  * tcgen05.mma M=128 reaches the full 8192 FLOP/clk/SM only for N >= 128 (N=64: ~48 clk
//    per K=16 step instead of 32; tools/mma_rate.cu), so S = Q K^T uses 128-key tiles.
//  * one CTA = one 128-row query tile of one head; 20 warps:
//      warps 0, 2  TMA producers: Q once; K (3 stages) and V (2 stages) in 128-key tiles
//      warp 1      TMEM allocator + tcgen05.mma issuer (warp-uniform loop, one lane issues)
//      warps 2-3   build the CTA's KV-tile schedule (tile kinds) in shared memory first
//      warps 4-19  softmax + epilogue: warp w owns TMEM lanes 32*(w%4).. (32 query rows)
//                  and key columns 32*cg.. of the tile, cg = (w-4)/4; the four warps of a
//                  lane quadrant exchange their row maxima through shared memory.
//  * TMEM (512 cols): O [0,128), S double buffer [128,256) [256,384), P (bf16) double
//    buffer [384,448) [448,512).  The MMA warp issues S(j+2) = Q K_{j+2}^T as soon as the
//    softmax warps have copied S(j) to registers, and O += P(j) V_j once P(j) is in TMEM,
//    so the tensor core computes scores two tiles ahead of the exponentials; P is the A
//    operand of PV straight from TMEM.
//  * four softmax warps per SMSP keep MUFU / FMA / issue busy (two per SMSP left them
//    latency-bound); packed fp32x2 FFMA2/FADD2; 3/8 of the exponentials run as a cubic
//    on the FMA pipe (rel. error 7.5e-5 << bf16's 2^-9) to relieve MUFU.
//  * lazy rescaling: the running max only moves when it grows by > 8 (log2 units); O is
//    rescaled in TMEM after PV(j-1) completed.
//  * masks from segment descriptors: empty tiles are skipped, full tiles run mask-free,
//    only diagonal / ragged tiles evaluate per-element positions.
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

constexpr int kThreads = 640;
constexpr int kSoftmaxWarps = 16;
constexpr int BM = 128;                 // query rows per CTA (TMEM lanes)
constexpr int BN = 128;                 // KV rows per tile
constexpr int kBox = 128 * 128;         // TMA box: 128 rows x 64 bf16 (128-byte swizzle rows)
constexpr int kSchedMax = 8192;         // KV tiles per launch (1M keys)

template <int HD>
struct Layout {
    static constexpr int NBOX = HD / 64;
    static constexpr int TILE = kBox * NBOX;  // one 128-row tile of Q, K or V
    static constexpr int KST = 3, VST = 2;
    static constexpr int OFF_Q = 0;
    static constexpr int OFF_K = OFF_Q + TILE;
    static constexpr int OFF_V = OFF_K + KST * TILE;
    static constexpr int OFF_RED = OFF_V + VST * TILE;  // [2 parity][4 quad][32 lanes][4 cg] float
    static constexpr int OFF_BAR = OFF_RED + 2 * 4 * 4 * 32 * 4;
    // q_full, k_full[KST], k_empty[KST], v_full[VST], v_empty[VST],
    // s_full[2], s_free[2], p_full[2], p_free[2], o_full
    static constexpr int B_Q = 0, B_KF = 1, B_KE = B_KF + KST, B_VF = B_KE + KST, B_VE = B_VF + VST,
                         B_SF = B_VE + VST, B_SE = B_SF + 2, B_PF = B_SE + 2, B_PE = B_PF + 2, B_O = B_PE + 2,
                         NBAR = B_O + 1;
    static constexpr int OFF_TMEM_SLOT = OFF_BAR + NBAR * 8;
    static constexpr int OFF_JR = OFF_TMEM_SLOT + 16;   // used-tile range: 2 x (min, max+1)
    static constexpr int OFF_SCHED = OFF_JR + 16;
    static constexpr int SMEM = OFF_SCHED + kSchedMax + 1024;  // + alignment slack
};

constexpr uint32_t COL_O = 0, COL_S = 128, COL_P = 384;  // S buffer b at COL_S + 128 b, P at COL_P + 64 b

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

__device__ __forceinline__ void named_bar_sync(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

template <int HD>
__global__ void __launch_bounds__(kThreads, 1)
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
    float* red = reinterpret_cast<float*>(smem + L::OFF_RED);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const cdsp_segments& sg = p.seg;

    // ---- work unit: head-major (the ~148 CTAs in flight share one head's K/V, which stays
    // L2-resident; head-minor order streamed all heads' K/V from DRAM ~40x over), heavy row
    // blocks first within a head (causal work grows with the row index)
    const int head = static_cast<int>(blockIdx.x) / p.n_rb;
    const int rb = p.n_rb - 1 - static_cast<int>(blockIdx.x) % p.n_rb;
    const int kvh = head / p.g;
    const int64_t row0 = static_cast<int64_t>(rb) * BM;
    const int n_kv_tiles = static_cast<int>((sg.nkv + BN - 1) / BN);

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
        for (int b = 0; b < 2; ++b) {
            mbar_init(bar(L::B_SF + b), 1);
            mbar_init(bar(L::B_SE + b), kSoftmaxWarps);
            mbar_init(bar(L::B_PF + b), kSoftmaxWarps);
            mbar_init(bar(L::B_PE + b), 1);
        }
        mbar_init(bar(L::B_O), 1);
        fence_barrier_init();
        tma_prefetch_desc(&tm_q);
        tma_prefetch_desc(&tm_k);
        tma_prefetch_desc(&tm_v);
        // Q does not depend on the schedule: start its load now
        mbar_expect_tx(bar(L::B_Q), L::TILE);
        for (int b = 0; b < L::NBOX; ++b)
            tma_load_3d(sQ + b * kBox, &tm_q, bar(L::B_Q), b * 64, head, static_cast<int>(row0));
    } else if (warp == 1) {
        tmem_alloc(smem_u32(tmem_slot), 512);
        tmem_relinquish();
    } else if (warp == 2 || warp == 3) {
        // KV-tile schedule: sched[j] = tile kind (0 = skip)
        int64_t qlo, qhi;
        bool qany;
        seg_qrange(sg, row0, row0 + BM, qlo, qhi, qany);
        int jmin = INT_MAX, jmax = 0;
        for (int j = (warp - 2) * 32 + lane; j < n_kv_tiles; j += 64) {
            const int k = seg_tile_kind(sg, qany, qlo, qhi, static_cast<int64_t>(j) * BN, BN);
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
            reinterpret_cast<int*>(smem + L::OFF_JR)[2 * (warp - 2)] = jmin;
            reinterpret_cast<int*>(smem + L::OFF_JR)[2 * (warp - 2) + 1] = jmax;
        }
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    // the used KV tiles lie in [j_lo, j_hi) (sched[j] == 0 marks skipped tiles inside it)
    const int* jr = reinterpret_cast<const int*>(smem + L::OFF_JR);
    const int j_lo = min(jr[0], jr[2]), j_hi = max(jr[1], jr[3]);
    if (threadIdx.x == 0) CTA_STAMP(4);

    if (warp == 0 || warp == 2) {
        // ======== TMA producers: warp 0 streams K, warp 2 streams V (independent rings, so a
        // K load never waits behind a V stage; one lane issues, the warp runs the loop) ========
        const bool is_k = warp == 0;
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
    } else if (warp == 1) {
        // ================= MMA issuer (warp-uniform loop, one lane issues) =================
        constexpr uint32_t idesc_qk = idesc_bf16_f32(BM, BN, false, false);
        constexpr uint32_t idesc_pv = idesc_bf16_f32(BM, HD, false, true);
        const uint64_t dq = umma_desc_sw128(sQ, 16, 1024);
        const uint64_t dk0 = umma_desc_sw128(sK, 16, 1024);
        const uint64_t dv0 = umma_desc_sw128(sV, kBox, 1024);
        // S(b) = Q K^T: M=128, N=128, K=HD in steps of 16 (32 B inside a 128-B swizzle row)
        auto issue_qk = [&](int ks, int b) {
            const uint64_t dk = dk0 + static_cast<uint64_t>((ks * L::TILE) >> 4);
#pragma unroll
            for (int kk = 0; kk < HD / 16; ++kk) {
                const uint64_t off = static_cast<uint64_t>(((kk / 4) * kBox + (kk % 4) * 32) >> 4);
                mma_ss(tmem + COL_S + 128 * b, dq + off, dk + off, idesc_qk, kk > 0 ? 1u : 0u);
            }
        };
        // O += P(b) V: M=128, N=HD, K=128 keys in steps of 16 (V rows, 2048 B)
        auto issue_pv = [&](int vs, int b, bool acc) {
            const uint64_t dv = dv0 + static_cast<uint64_t>((vs * L::TILE) >> 4);
#pragma unroll
            for (int kk = 0; kk < BN / 16; ++kk)
                mma_ts(tmem + COL_O, tmem + COL_P + 64 * b + kk * 8, dv + static_cast<uint64_t>((kk * 16 * 128) >> 4),
                       idesc_pv, (acc || kk > 0) ? 1u : 0u);
        };
        int n_used = 0;
        for (int j = j_lo; j < j_hi; ++j) n_used += sched[j] != 0;
        mbar_wait(bar(L::B_Q), 0);
        tc_fence_after();
        for (int it = 0; it < 2 && it < n_used; ++it) {  // prologue: S(0), S(1)
            mbar_wait(bar(L::B_KF + it), 0);
            tc_fence_after();
            if (elect_one()) {
                issue_qk(it, it);
                mma_commit(bar(L::B_SF + it));
                mma_commit(bar(L::B_KE + it));
            }
            __syncwarp();
        }
        for (int it = 0; it < n_used; ++it) {
            const int b = it & 1;
            const uint32_t ph = (it >> 1) & 1;
            if (it + 2 < n_used) {  // scores two tiles ahead, once softmax has read S(it)
                const int ks = (it + 2) % L::KST;
                mbar_wait(bar(L::B_SE + b), ph);
                mbar_wait(bar(L::B_KF + ks), ((it + 2) / L::KST) & 1);
                tc_fence_after();
                if (elect_one()) {
                    KTRACE(8, it);
                    issue_qk(ks, b);
                    mma_commit(bar(L::B_SF + b));
                    mma_commit(bar(L::B_KE + ks));
                    KTRACE(9, it);
                }
                __syncwarp();
            }
            const int vs = it % L::VST;
            mbar_wait(bar(L::B_VF + vs), (it / L::VST) & 1);
            mbar_wait(bar(L::B_PF + b), ph);
            tc_fence_after();
            if (elect_one()) {
                KTRACE(10, it);
                issue_pv(vs, b, it > 0);
                mma_commit(bar(L::B_PE + b));
                mma_commit(bar(L::B_VE + vs));
                if (it == n_used - 1) mma_commit(bar(L::B_O));
                KTRACE(11, it);
            }
            __syncwarp();
        }
    } else if (warp >= 4) {
        // ================= softmax + epilogue =================
        const int quad = warp & 3;       // TMEM lane quadrant: query rows 32*quad ..
        const int cg = (warp - 4) >> 2;  // key columns 32*cg .. of each S tile; O columns 32*cg ..
        const int r = quad * 32 + lane;
        const int64_t row = row0 + r;
        const bool row_ok = row < sg.nq;
        const int64_t my_qpos = row_ok ? seg_qpos(sg, row) : INT64_MAX;
        const uint32_t lane_off = static_cast<uint32_t>(quad * 32) << 16;
        const uint32_t tS = tmem + lane_off + COL_S + 32 * cg;
        const uint32_t tP = tmem + lane_off + COL_P + 16 * cg;
        const uint32_t tO = tmem + lane_off + COL_O + 32 * cg;
        const bool owns_o = cg * 32 < HD;  // HD = 64: column groups 2, 3 own no O columns
        const float sl2 = p.scale_log2;
        float m = -INFINITY;
        float2 lacc = make_float2(0.f, 0.f);
        // mask (diagonal / ragged tiles) and this warp's 32-column row max of one S tile
        auto mask_max = [&](uint32_t (&sv)[32], int j, int kind) {
            if (kind == TILE_PARTIAL) {
                const int64_t c0 = static_cast<int64_t>(j) * BN + 32 * cg;
#pragma unroll
                for (int i = 0; i < 32; ++i)
                    if (!seg_visible(sg, c0 + i, my_qpos)) sv[i] = __float_as_uint(-INFINITY);
            }
            float mx0 = -INFINITY, mx1 = -INFINITY, mx2 = -INFINITY, mx3 = -INFINITY;
#pragma unroll
            for (int i = 0; i < 32; i += 4) {
                mx0 = fmaxf(mx0, __uint_as_float(sv[i]));
                mx1 = fmaxf(mx1, __uint_as_float(sv[i + 1]));
                mx2 = fmaxf(mx2, __uint_as_float(sv[i + 2]));
                mx3 = fmaxf(mx3, __uint_as_float(sv[i + 3]));
            }
            return fmaxf(fmaxf(mx0, mx1), fmaxf(mx2, mx3));
        };
        // row max over the four column groups of this lane quadrant (parity-double-buffered)
        auto exchange_max = [&](float lmx, int parity) {
            float* rq = red + ((parity * 4 + quad) * 32 + lane) * 4;
            rq[cg] = lmx;
            named_bar_sync(1 + quad, 128);
            const float4 m4 = *reinterpret_cast<const float4*>(rq);
            return fmaxf(fmaxf(m4.x, m4.y), fmaxf(m4.z, m4.w));
        };
        int it = 0;
        for (int j = j_lo; j < j_hi; ++j) {
            const int kind = sched[j];
            if (kind == 0) continue;
            const int b = it & 1;
            const uint32_t ph = (it >> 1) & 1;
            uint32_t s[32];
            mbar_wait(bar(L::B_SF + b), ph);
            if (lane == 0 && (warp == 4 || warp == 19)) KTRACE(warp == 4 ? 0 : 4, it);
            tc_fence_after();
            tmem_ld32(tS + 128 * b, s);
            tc_wait_ld_regs(s);
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(bar(L::B_SE + b));  // S(b) may now be overwritten
            if (threadIdx.x == 128 && it == 0) CTA_STAMP(5);
            const float mx = exchange_max(mask_max(s, j, kind), it & 1);
            if (lane == 0 && warp == 4) KTRACE(1, it);
            const float m_new = fmaxf(m, mx * sl2);
            const bool need = m_new > m + 8.0f;
            if (__any_sync(0xFFFFFFFFu, need)) {
                const float alpha = need ? ex2(m - m_new) : 1.0f;
                if (need) {
                    lacc.x *= alpha;
                    lacc.y *= alpha;
                    m = m_new;
                }
                if (it > 0 && owns_o) {  // O holds PV up to it-1: wait for it, rescale 32 columns
                    mbar_wait(bar(L::B_PE + (b ^ 1)), ((it - 1) >> 1) & 1);
                    tc_fence_after();
                    uint32_t o[32];
                    tmem_ld32(tO, o);
                    tc_wait_ld_regs(o);
#pragma unroll
                    for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
                    tmem_st32(tO, o);
                }
            }
            const float m_use = (m == -INFINITY) ? 0.f : m;
            const float2 sc = make_float2(sl2, sl2), nm = make_float2(-m_use, -m_use);
            uint32_t pk[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                const float2 x = ffma2(make_float2(__uint_as_float(s[2 * i]), __uint_as_float(s[2 * i + 1])), sc, nm);
                float2 pp;
                if ((CDSP_EMU_MASK >> (i % 8)) & 1) {  // pairs on the FMA pipe (default 3/8: pairs 1, 4, 6 of 8)
                    pp = ex2_fma2(x);
                } else {
                    pp.x = ex2(x.x);
                    pp.y = ex2(x.y);
                }
                lacc = fadd2(lacc, pp);
                pk[i] = pack_bf16(pp.x, pp.y);
            }
            if (lane == 0 && warp == 4) KTRACE(2, it);
            if (it >= 2) {  // P(b) must have been consumed by PV(it-2)
                mbar_wait(bar(L::B_PE + b), ((it - 2) >> 1) & 1);
                tc_fence_after();
            }
            tmem_st16(tP + 64 * b, pk);
            tc_wait_st();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(bar(L::B_PF + b));
            if (lane == 0 && (warp == 4 || warp == 19)) KTRACE(warp == 4 ? 3 : 5, it);
            ++it;
        }

        // ---------------- epilogue: normalise, then write / LSE-merge (R3) ----------------
        const int n_used = it;
        if (threadIdx.x == 128) CTA_STAMP(6);
        if (n_used > 0) {
            mbar_wait(bar(L::B_O), 0);
            tc_fence_after();
        }
        // row sum over the four column groups (all four hold the same running max); the
        // exchange buffer of parity n_used is free: every warp of the quadrant passed the
        // last max exchange (parity n_used - 1) before writing here
        float* rs = red + (((n_used & 1) * 4 + quad) * 32 + lane) * 4;
        rs[cg] = lacc.x + lacc.y;
        named_bar_sync(1 + quad, 128);
        const float4 l4 = *reinterpret_cast<const float4*>(rs);
        const float l = (l4.x + l4.y) + (l4.z + l4.w);
        const float inv_l = l > 0.f ? 1.0f / l : 0.f;
        const float lse_b = l > 0.f ? (m + __log2f(l)) * 0.69314718055994530942f : -INFINITY;
        const int64_t nq = sg.nq;
        const size_t orow = (static_cast<size_t>(row_ok ? row : 0) * p.Hq + head) * HD + 32 * cg;
        float wa = 0.f, wb = 1.f, lse_out = lse_b;
        if (p.mode == CDSP_ATTN_MID || p.mode == CDSP_ATTN_LAST) {
            const float lse_a = row_ok ? p.lse_acc[static_cast<size_t>(head) * nq + row] : -INFINITY;
            merge_weights(lse_a, lse_b, wa, wb, lse_out);
        }
        const float sbw = wb * inv_l;
        uint32_t o[32];
        if (n_used > 0 && owns_o) {
            tmem_ld32(tO, o);
            tc_wait_ld();
        } else {
#pragma unroll
            for (int i = 0; i < 32; ++i) o[i] = 0u;
        }
        if (row_ok && owns_o) {
            float v[32];
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(o[i]) * sbw;
            if (p.mode == CDSP_ATTN_MID || p.mode == CDSP_ATTN_LAST) {
                const float4* a4 = reinterpret_cast<const float4*>(p.o_acc + orow);
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
                float4* d4 = reinterpret_cast<float4*>(p.o_acc + orow);
#pragma unroll
                for (int i = 0; i < 8; ++i) d4[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
            } else {
                uint4* d4 = reinterpret_cast<uint4*>(p.out + orow);
#pragma unroll
                for (int i = 0; i < 4; ++i)
                    d4[i] = make_uint4(pack_bf16(v[8 * i + 0], v[8 * i + 1]), pack_bf16(v[8 * i + 2], v[8 * i + 3]),
                                       pack_bf16(v[8 * i + 4], v[8 * i + 5]), pack_bf16(v[8 * i + 6], v[8 * i + 7]));
            }
            if (cg == 0) {
                const size_t li = static_cast<size_t>(head) * nq + row;
                if (p.mode == CDSP_ATTN_FIRST || p.mode == CDSP_ATTN_MID) {
                    p.lse_acc[li] = lse_out;
                } else if (p.lse) {
                    p.lse[li] = lse_out;
                }
            }
        }
        if (threadIdx.x == 128) CTA_STAMP(7);
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
    if (warp == 1) {
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
