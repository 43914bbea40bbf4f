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
//    The issuing thread is paced by the tensor pipe (a group of 8 MMAs is accepted about
//    when the previous group drains), so the MMA order below is the execution order.
//  * MUFU.EX2 issues 16 lanes/clk/SM (tools/exp_rate.cu): the 16384 exponentials of a
//    128x128 tile take 1024 clk, exactly the two MMAs of that tile, and TMEM reads run at
//    ~64 B/clk per SM sub-partition (64 KB of S: ~256 clk).  The softmax of one tile is
//    therefore longer than its MMAs; it must not sit on the tensor pipe's critical path.
//  * one CTA = one 128-row query tile of one head, 11 warps:
//      warps 0-3   softmax group 0: KV tiles 0, 2, 4, ... of the schedule
//      warps 4-7   softmax group 1: KV tiles 1, 3, 5, ...
//                  (warp w owns TMEM lanes 32*(w%4).., one thread = one query row holding
//                  all 128 scores of the tile in registers)
//      warp 8      TMA producer: Q once, then K tiles (3 stages)
//      warp 9      TMA producer: V tiles (2 stages)
//      warp 10     TMEM allocator + tcgen05.mma issuer (warp-uniform loop, one lane issues)
//  * TMEM (512 cols): O [0,128), S/P triple buffer [128,256) [256,384) [384,512).  P (bf16)
//    is written over its own S columns and is the A operand of PV straight from TMEM.  The
//    MMA order is S(0) S(1) S(2) | PV(0) S(3) | PV(1) S(4) | ...: S(n+3) reuses the buffer
//    of P(n) right after PV(n) (same in-order pipe), so scores are always two tiles ahead
//    and the two softmax groups overlap each other's exponentials.
//  * the only serial link between consecutive tiles is the running row max m (online
//    softmax): a group takes the row max of its own tile first, then m(n-1) from the other
//    group through shared memory, publishes m(n) and only then runs the exponentials.
//    Each group keeps its own row sum l (rescaled whenever m moves); the two are added in
//    the epilogue.  Lazy rescaling: m only moves when it grows by > 8 (log2 units); O is
//    then rescaled in TMEM after PV(n-1) completed and before m(n) is published.
//  * 1/8 of the exponentials run as a cubic on the FMA pipe (rel. error 7.5e-5, far below
//    bf16's 2^-9), packed fp32x2 FFMA2/FADD2.  Under sustained load the B200 sits at its
//    ~1000 W cap (SM clock ~1.5 GHz, tools/clock_probe.py), so energy per tile matters as much
//    as clocks per tile: 1/8 measured best sustained (1/4: -3.5%, 3/8: -3%, none: -1%).
//  * one score tile is 128 fp32 registers; holding it whole spilled loop state whose reloads
//    queue behind MUFU traffic, so a thread keeps 64 scores: columns 64-127 are read for the
//    row max, 0-63 for max + exponentials, and 64-127 again for theirs.
//  * masks from segment descriptors: empty tiles are skipped, full tiles run mask-free,
//    diagonal / ragged tiles build per-row 32-bit column masks from the three visible
//    intervals (history, segment 0, segment 1).
#include <cuda.h>
#include <cuda_bf16.h>

#include <climits>
#include <cstdio>
#include <cstdlib>

#include "attn_common.cuh"
#include "common.cuh"
#include "internal.h"
#include "ptx.cuh"

// MMA issuer's barrier waits: spin (lowest latency) or sleep on the phase (frees issue slots
// for the softmax warps sharing its SMSP)
#ifndef CDSP_MMA_SPIN
#define CDSP_MMA_SPIN 0
#endif
#if CDSP_MMA_SPIN
#define MMA_WAIT mbar_wait_spin
#else
#define MMA_WAIT mbar_wait
#endif

#ifndef CDSP_VST  // V shared-memory stages (K has one per S buffer)
#define CDSP_VST 2
#endif

#ifndef CDSP_EMU_MASK
#define CDSP_EMU_MASK 0x02
#endif

namespace cdsp {
using namespace ptx;

namespace {

constexpr int kThreads = 352;           // 11 warps
constexpr int BM = 128;                 // query rows per CTA (TMEM lanes)
constexpr int BN = 128;                 // KV rows per tile
constexpr int NSB = 3;                  // S/P buffers in TMEM
constexpr int kBox = 128 * 128;         // TMA box: 128 rows x 64 bf16 (128-byte swizzle rows)
constexpr int kSchedMax = 8192;         // KV tiles per launch (1M keys)
constexpr int W_K = 8, W_V = 9, W_MMA = 10;
constexpr int kSchedWarps = 8;          // warps 0-7 classify the KV tiles at setup

template <int HD>
struct Layout {
    static constexpr int NBOX = HD / 64;
    static constexpr int TILE = kBox * NBOX;  // one 128-row tile of Q, K or V
    static constexpr int KST = 3, VST = CDSP_VST;  // KST == NSB: K stage n%3 is free once S(n) is
    static constexpr int OFF_Q = 0;
    static constexpr int OFF_K = OFF_Q + TILE;
    static constexpr int OFF_V = OFF_K + KST * TILE;
    static constexpr int OFF_M = OFF_V + VST * TILE;       // running row max m(n): [2 parity][128] float
    static constexpr int OFF_L = OFF_M + 2 * BM * 4;       // epilogue: per-group (m_used, l) [2][128] float2
    static constexpr int OFF_QP = OFF_L + 2 * BM * 8;      // query position per row: [128] int64
    static constexpr int OFF_BAR = OFF_QP + BM * 8;
    // q_full, k_full[KST], v_full[VST], v_empty[VST], s_full[NSB], p_full[NSB], o_full.
    // (m(n) goes from one softmax group to the other through named barriers 2, 3.)  Every tcgen05.commit costs the tensor pipe ~30 clk (tools/mma_pattern.cu), so
    // each MMA group commits once: s_full[b] (S(n) done) also frees K stage n % 3, and
    // v_empty[s] (PV(n) done) also tells a rescaling softmax group that O is stable.
    static constexpr int B_Q = 0, B_KF = 1, B_VF = B_KF + KST, B_VE = B_VF + VST, B_SF = B_VE + VST,
                         B_PF = B_SF + NSB, B_OF = B_PF + NSB, B_ACC = B_OF + 1, NBAR = B_ACC + 1;
    static_assert(KST == NSB, "K stages are released through s_full");
    static constexpr int OFF_TMEM_SLOT = OFF_BAR + NBAR * 8;
    static constexpr int OFF_JR = OFF_TMEM_SLOT + 16;   // used-tile range per setup warp: (min, max+1)
    static constexpr int OFF_SCHED = OFF_JR + 12 * kSchedWarps;
    static constexpr int SMEM = OFF_SCHED + kSchedMax + 1024;  // + alignment slack
};

constexpr uint32_t COL_O = 0;
__host__ __device__ constexpr uint32_t col_s(int b) { return 128u + 128u * b; }

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
__device__ __forceinline__ void named_bar_arrive(int id, int nthreads) {
    asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
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
__device__ __forceinline__ void reg_tie16(uint32_t* r) {
    asm volatile(""
                 : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]),
                   "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]), "+r"(r[14]),
                   "+r"(r[15]));
}
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t (&r)[8]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(r[0]),
                 "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
                 : "memory");
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

// Mask columns [col0, col0 + 32*NW) of a partial tile (s[0] = column col0): the KV rows of
// tile j visible to a query at position qpos are the union of [0, b0) (history), [a1, b1)
// (segment 0 rows with pos <= qpos) and [a2, b2) (segment 1 rows with pos <= qpos),
// tile-relative — seg_visible() written as intervals.
template <int NW>
__device__ __forceinline__ void mask_cols(uint32_t* s, const cdsp_segments& sg, int j, int64_t qpos, int col0) {
    asm volatile("" : "+l"(qpos));  // keep this arithmetic on the (rare) partial-tile path
    const int64_t c0 = static_cast<int64_t>(j) * BN;
    const int nk = clamp_bn(sg.nkv - c0);
    const int h = clamp_bn(sg.kv_hist - c0);
    const int64_t e0abs = sg.kv_hist + sg.kv_len0;
    const int e0 = clamp_bn(e0abs - c0);
    // rows of segment 0 / 1 with position <= qpos: floor((qpos - pos0) / st) + 1 (0 if negative)
    int64_t n0 = qpos - sg.kv_pos0 + 1, n1 = qpos - sg.kv_pos1 + 1;
    if (sg.pos_stride != 1) {
        n0 = n0 > 0 ? (n0 - 1) / sg.pos_stride + 1 : 0;
        n1 = n1 > 0 ? (n1 - 1) / sg.pos_stride + 1 : 0;
    }
    const int lim0 = clamp_bn(n0 + sg.kv_hist - c0);
    const int lim1 = clamp_bn(n1 + e0abs - c0);
    const int b0 = min(h, nk);
    const int a1 = h, b1 = min(min(e0, lim0), nk);
    const int a2 = e0, b2 = min(nk, lim1);
#pragma unroll
    for (int w = 0; w < NW; ++w) {
        const int base = col0 + 32 * w;
        const uint32_t mk = range_bits(0, b0, base) | range_bits(a1, b1, base) | range_bits(a2, b2, base);
#pragma unroll
        for (int i = 0; i < 32; ++i)
            if (!((mk >> i) & 1u)) s[32 * w + i] = __float_as_uint(-INFINITY);
    }
}

__device__ __forceinline__ float max64(const uint32_t* s) {
    float a[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = fmaxf(__uint_as_float(s[2 * k]), __uint_as_float(s[2 * k + 1]));
#pragma unroll
    for (int i = 16; i < 64; i += 16)
#pragma unroll
        for (int k = 0; k < 8; ++k) a[k] = fmaxf(a[k], fmaxf(__uint_as_float(s[i + 2 * k]), __uint_as_float(s[i + 2 * k + 1])));
    return fmaxf(fmaxf(fmaxf(a[0], a[1]), fmaxf(a[2], a[3])), fmaxf(fmaxf(a[4], a[5]), fmaxf(a[6], a[7])));
}

// p = 2^(s*sl2 - m) for 32 scores -> 16 bf16 pairs stored to TMEM columns tP .. tP+15 (two
// tcgen05.st x8); row sum accumulated in lacc.  Pairs selected by CDSP_EMU_MASK run on the FMA pipe.
__device__ __forceinline__ void exp32_store(const uint32_t* s, float2 sc, float2 nm, float2& lacc, uint32_t tP) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        uint32_t pk[8];
#pragma unroll
        for (int ii = 0; ii < 8; ++ii) {
            const int i = 8 * h + ii;
            const float2 x = ffma2(make_float2(__uint_as_float(s[2 * i]), __uint_as_float(s[2 * i + 1])), sc, nm);
            float2 pp;
            if ((CDSP_EMU_MASK >> (i % 8)) & 1) {
                pp = ex2_fma2(x);
            } else {
                pp.x = ex2(x.x);
                pp.y = ex2(x.y);
            }
            lacc = fadd2(lacc, pp);
            pk[ii] = pack_bf16(pp.x, pp.y);
        }
        tmem_st8(tP + 8 * h, pk);
    }
}

template <int HD>
__global__ void __maxnreg__(168)
    attn_tc_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                   const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ CUtensorMap tm_acc,
                   const __grid_constant__ CUtensorMap tm_out, const TcParams p) {
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

    // ---- setup
    if (warp == W_K) {
        if (lane == 0) {
            mbar_init(bar(L::B_Q), 1);
            for (int i = 0; i < L::KST; ++i) mbar_init(bar(L::B_KF + i), 1);
            for (int i = 0; i < L::VST; ++i) {
                mbar_init(bar(L::B_VF + i), 1);
                mbar_init(bar(L::B_VE + i), 1);
            }
            for (int b = 0; b < NSB; ++b) {
                mbar_init(bar(L::B_SF + b), 1);
                mbar_init(bar(L::B_PF + b), 4);
            }
            mbar_init(bar(L::B_OF), 1);
            mbar_init(bar(L::B_ACC), 1);
            fence_barrier_init();
            tma_prefetch_desc(&tm_q);
            tma_prefetch_desc(&tm_k);
            tma_prefetch_desc(&tm_v);
            if constexpr (HD == 128) {
                tma_prefetch_desc(&tm_acc);
                tma_prefetch_desc(&tm_out);
            }
            // Q does not depend on the schedule: start its load now
            mbar_expect_tx(bar(L::B_Q), L::TILE);
            for (int b = 0; b < L::NBOX; ++b)
                tma_load_3d(sQ + b * kBox, &tm_q, bar(L::B_Q), b * 64, head, static_cast<int>(row0));
        }
    } else if (warp == W_MMA) {
        tmem_alloc(smem_u32(tmem_slot), 512);
        tmem_relinquish();
    } else if (warp < kSchedWarps) {
        // KV-tile schedule: sched[j] = tile kind (0 = skip)
        int64_t qlo, qhi;
        bool qany;
        seg_qrange(sg, row0, row0 + BM, qlo, qhi, qany);
        int jmin = INT_MAX, jmax = 0, cnt = 0;
        for (int j = warp * 32 + lane; j < n_kv_tiles; j += kSchedWarps * 32) {
            const int k = seg_tile_kind(sg, qany, qlo, qhi, static_cast<int64_t>(j) * BN, BN);
            sched[j] = static_cast<uint8_t>(k);
            if (k != 0) {
                jmin = min(jmin, j);
                jmax = max(jmax, j + 1);
                ++cnt;
            }
        }
        for (int o = 16; o > 0; o >>= 1) {
            jmin = min(jmin, __shfl_xor_sync(0xFFFFFFFFu, jmin, o));
            jmax = max(jmax, __shfl_xor_sync(0xFFFFFFFFu, jmax, o));
            cnt += __shfl_xor_sync(0xFFFFFFFFu, cnt, o);
        }
        if (lane == 0) {
            reinterpret_cast<int*>(smem + L::OFF_JR)[3 * warp] = jmin;
            reinterpret_cast<int*>(smem + L::OFF_JR)[3 * warp + 1] = jmax;
            reinterpret_cast<int*>(smem + L::OFF_JR)[3 * warp + 2] = cnt;
        }
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    // the n_used used KV tiles lie in [j_lo, j_hi) (sched[j] == 0 marks skipped tiles inside)
    int j_lo = INT_MAX, j_hi = 0, n_used = 0;
    {
        const int* jr = reinterpret_cast<const int*>(smem + L::OFF_JR);
#pragma unroll
        for (int w = 0; w < kSchedWarps; ++w) {
            j_lo = min(j_lo, jr[3 * w]);
            j_hi = max(j_hi, jr[3 * w + 1]);
            n_used += jr[3 * w + 2];
        }
    }
    if (threadIdx.x == 0) CTA_STAMP(4);

    if (warp == W_K || warp == W_V) {
        // ======== TMA producers: K and V in independent rings (a K load never waits behind a
        // V stage); one lane issues, the warp runs the loop ========
        const bool is_k = warp == W_K;
        const int nst = is_k ? L::KST : L::VST;
        const uint32_t s0 = is_k ? sK : sV;
        const int bfull = is_k ? L::B_KF : L::B_VF, bempty = is_k ? L::B_SF : L::B_VE;
        const void* map = is_k ? static_cast<const void*>(&tm_k) : static_cast<const void*>(&tm_v);
        const uint64_t pol_kv = policy_evict_last();
        int it = 0;
        for (int j = j_lo; j < j_hi; ++j) {
            if (sched[j] == 0) continue;
            const int st = it % nst;
            // stage st last held tile it - nst: free once S(it - nst) (K) / PV(it - nst) (V) is done
            if (it >= nst) mbar_wait(bar(bempty + st), ((it - nst) / nst) & 1);
            if (elect_one()) {
                mbar_expect_tx(bar(bfull + st), L::TILE);
                for (int b = 0; b < L::NBOX; ++b)
                    tma_load_3d_hint(s0 + st * L::TILE + b * kBox, map, bar(bfull + st), b * 64, kvh, j * BN, pol_kv);
            }
            __syncwarp();
            ++it;
        }
        if constexpr (HD == 128) {
            // merge modes: once the last S = Q K^T has read the K stages, stage this tile's
            // fp32 accumulator rows there (4 boxes of 128 rows x 32 columns, 128B-swizzled) for
            // the epilogue — under the tail of the main loop instead of after it
            if (is_k && (p.mode == CDSP_ATTN_MID || p.mode == CDSP_ATTN_LAST)) {
                if (it > 0) {
                    const int nl = it - 1;  // the last used tile's S buffer / phase
                    mbar_wait(bar(L::B_SF + nl % NSB), (nl / NSB) & 1);
                }
                if (elect_one()) {
                    mbar_expect_tx(bar(L::B_ACC), BM * HD * 4);
                    for (int b = 0; b < HD / 32; ++b)
                        tma_load_3d(sK + b * (BM * 128), &tm_acc, bar(L::B_ACC), b * 32, head, static_cast<int>(row0));
                }
                __syncwarp();
            }
        }
    } else if (warp == W_MMA) {
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
                mma_ss(tmem + col_s(b), dq + off, dk + off, idesc_qk, kk > 0 ? 1u : 0u);
            }
        };
        // O += P(b) V: M=128, N=HD, K=128 keys in steps of 16 (V rows, 2048 B); P(b) is bf16
        // in the S(b) columns (8 TMEM columns per 16 keys)
        auto issue_pv = [&](int vs, int b, bool acc) {
            const uint64_t dv = dv0 + static_cast<uint64_t>((vs * L::TILE) >> 4);
#pragma unroll
            for (int kk = 0; kk < BN / 16; ++kk)
                mma_ts(tmem + COL_O, tmem + col_s(b) + kk * 8, dv + static_cast<uint64_t>((kk * 16 * 128) >> 4),
                       idesc_pv, (acc || kk > 0) ? 1u : 0u);
        };
        auto issue_s = [&](int n) {  // S(n) into buffer n % NSB; K stage n % KST
            const int ks = n % L::KST;
            MMA_WAIT(bar(L::B_KF + ks), (n / L::KST) & 1);
            tc_fence_after();
            if (elect_one()) {
                KTRACE(9, n);
                issue_qk(ks, n % NSB);
                mma_commit(bar(L::B_SF + n % NSB));  // S(n) ready; K stage ks free
            }
            __syncwarp();
        };
        if (n_used > 0) {
            MMA_WAIT(bar(L::B_Q), 0);
            for (int n = 0; n < NSB && n < n_used; ++n) issue_s(n);
        }
        for (int n = 0; n < n_used; ++n) {
            const int b = n % NSB, vs = n % L::VST;
            MMA_WAIT(bar(L::B_VF + vs), (n / L::VST) & 1);
            MMA_WAIT(bar(L::B_PF + b), (n / NSB) & 1);
            tc_fence_after();
            if (elect_one()) {
                KTRACE(8, n);
                issue_pv(vs, b, n > 0);
                mma_commit(bar(L::B_VE + vs));  // V stage free; O includes PV(n)
                if (n == n_used - 1) mma_commit(bar(L::B_OF));
            }
            __syncwarp();
            if (n + NSB < n_used) issue_s(n + NSB);  // into the buffer P(n) just left
        }
        if (n_used == 0) {
            if (elect_one()) mma_commit(bar(L::B_OF));
            __syncwarp();
        }
    } else if (warp < 8) {
        // ========= softmax group g (tiles n = g, g+2, ...): thread = one query row =========
        const int g = warp >> 2;
        const int quad = warp & 3;  // TMEM lane quadrant
        const int r = quad * 32 + lane;
        const int64_t row = row0 + r;
        const bool row_ok = row < sg.nq;
        // the row's query position is only needed on partial tiles: keep it out of registers
        int64_t* qpos_sh = reinterpret_cast<int64_t*>(smem + L::OFF_QP);
        if (g == 0) qpos_sh[r] = row_ok ? seg_qpos(sg, row) : (INT64_MAX >> 2);
        asm volatile("bar.sync 1, 256;" ::: "memory");
        const uint32_t lane_off = static_cast<uint32_t>(quad * 32) << 16;
        const uint32_t tO = tmem + lane_off + COL_O;
        float* msh = reinterpret_cast<float*>(smem + L::OFF_M);  // [2][BM]
        const float sl2 = p.scale_log2;
        float m = -INFINITY;       // m(n) of the last tile this thread has seen
        float m_used = -INFINITY;  // max that this group's l is relative to
        float2 lacc = make_float2(0.f, 0.f);
        // group g takes used tiles n = g, g+2, ...; jc = KV tile index of tile n
        auto next_used = [&](int jj) {
            ++jj;
            while (jj < j_hi && sched[jj] == 0) ++jj;
            return jj;
        };
        int jc = j_lo;
        if (g == 1 && n_used > 1) jc = next_used(jc);
        for (int n = g; n < n_used; n += 2, jc = next_used(next_used(jc))) {
            const int j = jc;
            const int kind = sched[j];
            const int b = n % NSB;
            const uint32_t tS = tmem + lane_off + col_s(b);
            if (lane == 0 && quad == 0) KTRACE(12 + g, n);
            mbar_wait(bar(L::B_SF + b), (n / NSB) & 1);
            if (lane == 0 && quad == 0) KTRACE(4 * g + 0, n);
            tc_fence_after();
#if defined(CDSP_DBG_SOFTMAX) && CDSP_DBG_SOFTMAX == 0
            // debug: MMA pipeline alone (no TMEM traffic from the softmax; results garbage)
            if (n > 0) named_bar_sync(2 + ((n - 1) & 1), 2 * BM);
            named_bar_arrive(2 + (n & 1), 2 * BM);
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(bar(L::B_PF + b));
            continue;
#endif
            // 64 score registers: columns 64-127 first (max only), then 0-63 (max, kept for the
            // exponentials); 64-127 are re-read from TMEM for their exponentials (P(n) only ever
            // overwrites S columns 0-63)
            uint32_t s[64];
            tmem_ld32p(tS + 64, s);
            tmem_ld32p(tS + 96, s + 32);
            tc_wait_ld();
            reg_tie32(s);
            reg_tie32(s + 32);
            if (threadIdx.x == 0 && n == 0) CTA_STAMP(5);
            const bool partial = kind == TILE_PARTIAL;
            if (partial) mask_cols<2>(s, sg, j, qpos_sh[r], 64);
            const float mx_hi = max64(s);
            tmem_ld32p(tS, s);
            tmem_ld32p(tS + 32, s + 32);
            tc_wait_ld();
            reg_tie32(s);
            reg_tie32(s + 32);
            if (partial) mask_cols<2>(s, sg, j, qpos_sh[r], 0);
            const float mx = fmaxf(mx_hi, max64(s)) * sl2;
            // ---- the serial link: m(n) = lazy max(m(n-1), rowmax(S(n))) ----
            if (n > 0) {  // m(n-1) from the other group (named barrier 2 + parity: 128 + 128 threads)
                named_bar_sync(2 + ((n - 1) & 1), 2 * BM);
                m = msh[((n - 1) & 1) * BM + r];
            }
            const bool need = mx > m + 8.0f;
            const float m_prev = m;
            if (need) m = mx;
            if (lane == 0 && quad == 0) KTRACE(4 * g + 1, n);
            // O holds PV up to n-1 relative to m(n-1): rescale it once PV(n-1) completed, before
            // m(n) is published (so no later PV can be issued meanwhile)
            if (n > 0 && __any_sync(0xFFFFFFFFu, need)) {
                mbar_wait(bar(L::B_VE + (n - 1) % L::VST), ((n - 1) / L::VST) & 1);  // PV(n-1) done
                tc_fence_after();
                const float alpha = need ? ex2(m_prev - m) : 1.0f;
#pragma unroll 1
                for (int c = 0; c < HD / 16; ++c) {
                    uint32_t o[16];
                    tmem_ld16(tO + 16 * c, o);
                    tc_wait_ld();
                    reg_tie16(o);
#pragma unroll
                    for (int i = 0; i < 16; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
                    tmem_st16(tO + 16 * c, o);
                }
            }
            msh[(n & 1) * BM + r] = m;
            __threadfence_block();
            named_bar_arrive(2 + (n & 1), 2 * BM);
#if defined(CDSP_DBG_SOFTMAX) && CDSP_DBG_SOFTMAX == 1
            // debug: S read + row max only, no exponentials / P stores
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(bar(L::B_PF + b));
            continue;
#endif
            // this group's row sum follows m
            if (m != m_used) {
                const float beta = ex2(m_used - m);  // m_used = -inf: l is 0 anyway
                lacc.x *= beta;
                lacc.y *= beta;
                m_used = m;
            }
            const float m_use = (m == -INFINITY) ? 0.f : m;
            const float2 sc = make_float2(sl2, sl2), nm = make_float2(-m_use, -m_use);
            // keys 0-63 from registers -> P columns 0-31; keys 64-127 re-read in two pieces,
            // each load in flight behind the previous piece's exponentials
            exp32_store(s, sc, nm, lacc, tS);
            tmem_ld32p(tS + 64, s);
            exp32_store(s + 32, sc, nm, lacc, tS + 16);
            tc_wait_ld();
            reg_tie32(s);
            tmem_ld32p(tS + 96, s + 32);
            if (partial) mask_cols<1>(s, sg, j, qpos_sh[r], 64);
            exp32_store(s, sc, nm, lacc, tS + 32);
            tc_wait_ld();
            reg_tie32(s + 32);
            if (partial) mask_cols<1>(s + 32, sg, j, qpos_sh[r], 96);
            exp32_store(s + 32, sc, nm, lacc, tS + 48);
            if (lane == 0 && quad == 0) KTRACE(4 * g + 2, n);
            tc_wait_st();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(bar(L::B_PF + b));
            if (lane == 0 && quad == 0) KTRACE(4 * g + 3, n);
        }

        // ---------------- epilogue: normalise, then write / LSE-merge (R3) ----------------
        if (threadIdx.x == 0) CTA_STAMP(6);
        // final m = m(n_used-1); combine the two groups' row sums relative to it
        float2* lsh = reinterpret_cast<float2*>(smem + L::OFF_L);  // [2][BM] (m_used, l)
        lsh[g * BM + r] = make_float2(m_used, lacc.x + lacc.y);
        if (n_used > 0 && ((n_used - 1) & 1) != g) {  // the other group made the last m: take it
            named_bar_sync(2 + ((n_used - 1) & 1), 2 * BM);  // (pairs with its last arrive)
            m = msh[((n_used - 1) & 1) * BM + r];
        }
        asm volatile("bar.sync 1, 256;" ::: "memory");  // both groups' (m_used, l) visible
        float l = 0.f;
#pragma unroll
        for (int gg = 0; gg < 2; ++gg) {
            const float2 ml = lsh[gg * BM + r];
            if (ml.y > 0.f) l += ml.y * ex2(ml.x - m);
        }
        mbar_wait(bar(L::B_OF), 0);
        tc_fence_after();
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
        if constexpr (HD == 128) {
            // Staged epilogue: thread = row, but global traffic goes through 128B-swizzled smem
            // tiles moved by TMA (a thread-per-row store touches 32 rows per warp instruction).
            // fp32 results (FIRST/MID) are written in place over the accumulator tile in the K
            // stages; bf16 results (ONLY/LAST) into the V stages.  Group g owns columns
            // [64 g, 64 g + 64): fp32 boxes 2g, 2g+1 (32 columns each), bf16 box g.
            if (merge) mbar_wait(bar(L::B_ACC), 0);  // accumulator tile landed (K warp's TMA)
            const uint32_t rsw = static_cast<uint32_t>(r & 7);
#pragma unroll
            for (int cc = 0; cc < 2; ++cc) {
                uint32_t o[32];
                if (n_used > 0) {
                    tmem_ld32p(tO + 32 * (2 * g + cc), o);
                    tc_wait_ld();
                    reg_tie32(o);
                } else {
#pragma unroll
                    for (int i = 0; i < 32; ++i) o[i] = 0u;
                }
                float v[32];
#pragma unroll
                for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(o[i]) * sbw;
                const uint32_t fbox = sK + static_cast<uint32_t>(2 * g + cc) * (BM * 128) + static_cast<uint32_t>(r) * 128;
                if (merge) {
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        float4 av;
                        asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];"
                                     : "=f"(av.x), "=f"(av.y), "=f"(av.z), "=f"(av.w)
                                     : "r"(fbox + ((j ^ rsw) << 4)));
                        v[4 * j + 0] = fmaf(wa, av.x, v[4 * j + 0]);
                        v[4 * j + 1] = fmaf(wa, av.y, v[4 * j + 1]);
                        v[4 * j + 2] = fmaf(wa, av.z, v[4 * j + 2]);
                        v[4 * j + 3] = fmaf(wa, av.w, v[4 * j + 3]);
                    }
                }
                if (to_acc) {
#pragma unroll
                    for (int j = 0; j < 8; ++j)
                        asm volatile("st.shared.v4.f32 [%0], {%1,%2,%3,%4};" ::"r"(fbox + ((j ^ rsw) << 4)),
                                     "f"(v[4 * j]), "f"(v[4 * j + 1]), "f"(v[4 * j + 2]), "f"(v[4 * j + 3])
                                     : "memory");
                } else {
                    const uint32_t hbox = sV + static_cast<uint32_t>(g) * (BM * 128) + static_cast<uint32_t>(r) * 128;
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const uint32_t ch = static_cast<uint32_t>(4 * cc + j);
                        asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(hbox + ((ch ^ rsw) << 4)),
                                     "r"(pack_bf16(v[8 * j + 0], v[8 * j + 1])), "r"(pack_bf16(v[8 * j + 2], v[8 * j + 3])),
                                     "r"(pack_bf16(v[8 * j + 4], v[8 * j + 5])), "r"(pack_bf16(v[8 * j + 6], v[8 * j + 7]))
                                     : "memory");
                    }
                }
            }
            fence_proxy_async_smem();
            named_bar_sync(4 + g, BM);  // this group's 128 rows are in smem
            if (threadIdx.x == static_cast<unsigned>(g * BM)) {
                if (to_acc) {
                    for (int cc = 0; cc < 2; ++cc)
                        tma_store_3d(&tm_acc, sK + static_cast<uint32_t>(2 * g + cc) * (BM * 128), 32 * (2 * g + cc), head,
                                     static_cast<int>(row0));
                } else {
                    tma_store_3d(&tm_out, sV + static_cast<uint32_t>(g) * (BM * 128), 64 * g, head, static_cast<int>(row0));
                }
                bulk_commit();
                bulk_wait_read0();  // smem stays valid until the store has read it
            }
        } else {
        // group g writes O columns [g*HD/2, (g+1)*HD/2)
#pragma unroll 1
        for (int c = g * (HD / 64); c < (g + 1) * (HD / 64); ++c) {
            uint32_t o[32];
            if (n_used > 0) {
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
                        const float4 av = a4[i];
                        v[4 * i + 0] = fmaf(wa, av.x, v[4 * i + 0]);
                        v[4 * i + 1] = fmaf(wa, av.y, v[4 * i + 1]);
                        v[4 * i + 2] = fmaf(wa, av.z, v[4 * i + 2]);
                        v[4 * i + 3] = fmaf(wa, av.w, v[4 * i + 3]);
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
        }  // HD != 128
        if (row_ok && g == 0) {
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
// fp32 [T, H, D], box = 128 rows x 1 head x 32 columns (128 B), 128-byte swizzle (epilogue staging).
cdsp_status make_map_f32(CUtensorMap* m, const void* base, int64_t T, int H, int D) {
    EncodeTiledFn enc = get_encode_fn();
    CDSP_REQUIRE(enc != nullptr, CDSP_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    CDSP_REQUIRE((reinterpret_cast<uintptr_t>(base) & 15u) == 0, CDSP_ERR_INVALID,
                 "TMA base pointer must be 16-byte aligned");
    cuuint64_t dims[3] = {static_cast<cuuint64_t>(D), static_cast<cuuint64_t>(H),
                          static_cast<cuuint64_t>(T > 0 ? T : 1)};
    cuuint64_t strides[2] = {static_cast<cuuint64_t>(D) * 4, static_cast<cuuint64_t>(H) * D * 4};
    cuuint32_t box[3] = {32, 1, 128};
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<void*>(base), dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    CDSP_REQUIRE(r == CUDA_SUCCESS, CDSP_ERR_CUDA, "cuTensorMapEncodeTiled(f32) failed (%d)", static_cast<int>(r));
    return CDSP_OK;
}

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
    // epilogue maps (HD = 128): fp32 accumulators (FIRST/MID/LAST) and the bf16 output
    // (ONLY/LAST); a mode that does not use one gets a never-dereferenced stand-in
    CUtensorMap macc = mq, mout = mq;
    if (HD == 128 && a.seg.nq > 0) {
        if (a.mode != CDSP_ATTN_ONLY) CDSP_CHECK_STATUS(make_map_f32(&macc, a.o_acc, a.seg.nq, a.Hq, HD));
        if (a.mode == CDSP_ATTN_ONLY || a.mode == CDSP_ATTN_LAST)
            CDSP_CHECK_STATUS(make_map(&mout, a.out, a.seg.nq, a.Hq, HD));
    }
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
    attn_tc_kernel<HD><<<static_cast<unsigned>(grid), kThreads, Lt::SMEM, st>>>(mq, mk, mv, macc, mout, p);
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
