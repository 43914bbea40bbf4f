// attn_tc.cu — K*1: bf16 block attention for one ring step on sm_100a tensor cores.
//
// Computes, for a query shard and one KV block (history + a current-chunk shard), exact
// softmax attention under the position mask of attn_common.cuh, and writes or LSE-merges
// the result (cdsp_attn_mode).  This is the per-step compute of ring attention
// (§2.3: each instance "interact[s] local query tensors with full key-value
// tensors"), extended to historical tokens as Tetris does (§6: "we extend Flash
// Attention [7] to support zigzag ring attention for historical tokens").
//
// B200 design (not the paper's A100 FlashAttention-2), from measurements on the box (DESIGN.md
// 6.1 has the numbers and the tools):
//  * tcgen05.mma M=128 reaches the full 8192 FLOP/clk/SM only for N >= 128, so S = Q K^T uses
//    128-key tiles; a KV tile costs the tensor pipe 1024 clk (S and PV, 512 each).
//  * Supply, not math, bounds a 1-SM kernel: 64 KB of K+V per tile per SM from L2 capped the
//    MMA pipe at ~1373 clk/tile.  HD = 128 therefore runs as CTA PAIRS (cluster of 2,
//    tcgen05 cta_group::2, M = 256): each CTA holds its own 128 query rows (Q, S/P, O in its
//    TMEM) and half of every K tile (64 keys) and V tile (64 of 128 d columns); the even CTA
//    issues the MMAs, completions are multicast commits, both CTAs' TMA bytes and softmax
//    arrivals land on the even CTA's barriers.  HD = 64 (and CDSP_ATTN_1SM=1) run the same
//    code on one SM per unit (PAIR = false).
//  * Persistent: one CTA per SM, work units (a pair of 128-row blocks x one head) claimed from
//    an atomic counter, head-major and heaviest first; a scheduler warp publishes each unit's
//    compacted list of used KV tiles and loads its Q (double-buffered u_full / u_empty), cued
//    by the K producer a few tiles before the current unit's end.
//  * 12 warps: 0-3 and 4-7 two softmax groups (one thread = one query row = one TMEM lane)
//    taking alternate KV tiles; 8 TMA producer of K (3 stages); 9 TMA producer of V (3 stages
//    in PAIR); 10 TMEM allocator + MMA issuer; 11 unit scheduler + TMA producer of Q (2
//    buffers in PAIR).  3 warps per sub-partition x 168 registers.
//  * TMEM (512 cols): O [0,128), S/P triple buffer [128,256) [256,384) [384,512); P (bf16) is
//    written over its own S columns and is PV's A operand straight from TMEM.  MMA order
//    S(0) S(1) S(2) | PV(0) S(3) | PV(1) S(4) | ...: scores run two tiles ahead.
//  * The only serial link between consecutive tiles is the running row max m (online
//    softmax): a group reads its tile (all 128 scores in registers), takes m(n-1) from the
//    other group over a named barrier, publishes m(n) before its exponentials.  Lazy
//    rescaling: m moves only when it grows by > 8 (log2 units); O is then rescaled in TMEM
//    after PV(n-1) completed and before m(n) is published.  Each group keeps its own row sum.
//  * The softmax is bound by its instruction stream (~1340 clk/tile vs 1037 for the MMA pipe
//    alone): FMNMX3 row max, 1/8 of the exponentials as a cubic on the FMA pipe (rel. error
//    7.5e-5, far below bf16's 2^-9; same-box sweep 0 / 1/8 / 1/4 = 1313 / 1340 / 1267 TF/s).
//  * The group that computed a unit's last tile finishes the unit (the other hands over its
//    row sum and starts the next unit): O drained from TMEM in two 64-column halves, bf16
//    results TMA-stored from 128B-swizzled boxes, fp32 accumulators merged (R3) through
//    per-warp swizzled transposes (coalesced 512-byte warp transactions).
//  * MID / LAST launches are programmatic dependents of the previous launch (the next ring
//    step's main loop runs under this one's tail; the accumulator is touched after
//    griddepcontrol.wait).
//  * Masks from segment descriptors: empty tiles are skipped, full tiles run mask-free,
//    diagonal / ragged tiles build per-row 32-bit column masks from the three visible
//    intervals (history, segment 0, segment 1).
#include <cuda.h>
#include <cuda_bf16.h>

#include <climits>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

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

// unit scheduler: the next unit is claimed when the K producer is this many tiles from the end of
// the current one
#ifndef CDSP_PREP_LEAD
#define CDSP_PREP_LEAD 6
#endif
constexpr int kPrepLead = CDSP_PREP_LEAD;
#ifndef CDSP_VST  // V shared-memory stages (K has one per S buffer)
#define CDSP_VST 2
#endif

#ifndef CDSP_MAXNREG  // 12 warps: 3 per sub-partition x 168 regs x 32 lanes fills its 16K registers
#define CDSP_MAXNREG 168
#endif

#ifndef CDSP_FULL_ROW  // softmax holds the whole 128-score row (else two 64-score halves)
#define CDSP_FULL_ROW 1
#endif

#ifndef CDSP_EPI_WIDE  // FIRST / MID epilogue: 64 accumulator columns per L2 round trip
#define CDSP_EPI_WIDE 1
#endif

#ifndef CDSP_EPI_COALESCED  // fp32 accumulator epilogue through the warp-transpose tiles (PAIR)
#define CDSP_EPI_COALESCED 1
#endif

// Hand-over barriers (unit list / positions, row-sum slots): every lane arrives (1), so each
// lane's own shared-memory accesses are ordered by its own arrive — the happens-before
// compute-sanitizer's racecheck verifies — or lane 0 arrives after __syncwarp (0).
#ifndef CDSP_ALL_LANE_ARRIVE
#define CDSP_ALL_LANE_ARRIVE 1
#endif
#define ARRIVERS (CDSP_ALL_LANE_ARRIVE ? 32 : 1)
#define ARRIVE_LANE (CDSP_ALL_LANE_ARRIVE || lane == 0)

#ifndef CDSP_DBG_NO_KV  // debug probe (timing only, results garbage): 1 skip K tile loads, 2 skip V, 3 both
#define CDSP_DBG_NO_KV 0
#endif

#ifndef CDSP_KV_POLICY  // L2 policy of the K / V tile loads: 0 evict_last, 1 evict_normal, 2 evict_first
#define CDSP_KV_POLICY 0
#endif

#ifndef CDSP_EMU_MASK
#define CDSP_EMU_MASK 0x02
#endif

namespace cdsp {
using namespace ptx;

namespace {

// two softmax groups of 4 warps (a third group, 15 warps, was measured: not faster, the
// 128-register cap of 4 warps per sub-partition costs what the extra latency slack gains)
// softmax groups (warpgroups taking tiles n mod NG).  3 (with setmaxnreg: 12 x 152 registers) was
// measured slower: 1068 TF/s holding whole score rows (spills), 1264 / 1225 with 64-score halves
#ifndef CDSP_NGROUPS
#define CDSP_NGROUPS 2
#endif
constexpr int NG = CDSP_NGROUPS;
// CDSP_EPI_WARPS=1 (measured, not the default): a dedicated epilogue warpgroup finishes every
// unit (O drain, normalisation, output / accumulator writes), so both softmax groups run
// straight into the next unit.  Same box, 32K s=1: 1331 / 1316 vs 1337 / 1304 TF/s — the unit
// boundary is not what bounds the kernel (the softmax groups' per-tile stream is).  The
// CTA is 4 whole warpgroups (setmaxnreg acts per warpgroup; the fourth has one idle warp) and
// launches at 128 registers per thread, redistributed with setmaxnreg: softmax 168, epilogue
// 112, producers / MMA / idle 64 (8 x 168 + 4 x 112 + 4 x 64 = 16 x 128: an .inc beyond the
// CTA's pool would wait forever).  0: the group that computed a unit's last tile finishes it
// (round 1).
#ifndef CDSP_EPI_WARPS
#define CDSP_EPI_WARPS 0
#endif
constexpr int NEPI = CDSP_EPI_WARPS ? 4 : 0;
// register redistribution (setmaxnreg) whenever the CTA outgrows 12 warps at 168 registers:
// softmax / epilogue / producers+MMA+idle; 16 warps launched at 128 registers each
#define CDSP_REGSPLIT (CDSP_EPI_WARPS || CDSP_NGROUPS > 2)
constexpr int kThreads = 32 * (4 * NG + NEPI + 4);  // softmax, epilogue, K / V producers, MMA, scheduler
static_assert(!CDSP_REGSPLIT || kThreads == 512, "register split assumes 16 warps");
static_assert(NG == 2 || (NG == 3 && !CDSP_EPI_WARPS), "NG = 3 runs without the epilogue group");
#define CDSP_SOFTMAX_REGS (NG == 3 ? 152 : 168)
#define CDSP_PRODUCER_REGS (NG == 3 ? 56 : 64)
constexpr int BM = 128;                 // query rows per CTA (TMEM lanes)
constexpr int BN = 128;                 // KV rows per tile
constexpr int NSB = 3;                  // S/P buffers in TMEM
constexpr int kBox = 128 * 128;         // TMA box: 128 rows x 64 bf16 (128-byte swizzle rows)
constexpr int kSchedMax = 8192;         // KV tiles per launch (1M keys)
constexpr int kMaxBlk = CDSP_MAX_SP;    // KV blocks one launch walks (a rank's whole ring)
// roles are warpgroup-aligned (setmaxnreg acts per warpgroup): softmax 0..4NG-1, epilogue
// 4NG..4NG+3 (TMEM quadrants 0..3), then K producer, V producer, MMA
constexpr int W_EPI0 = 4 * NG;
constexpr int W_K = 4 * NG + NEPI, W_V = W_K + 1, W_MMA = W_K + 2, W_SCH = W_K + 3;

// PAIR: 2-SM variant (HD = 128).  A CTA pair (cluster of 2) runs M = 256 MMAs (cta_group::2):
// each CTA holds its own 128 query rows of Q and of S / P / O in its TMEM, and HALF of every
// K tile (64 keys) and V tile (64 of the 128 d columns) — so each SM streams 32 KB per KV tile
// from L2 instead of 64 KB.  The even CTA issues the MMAs; S / V / O completions are
// multicast to both CTAs' barriers, both CTAs' TMA bytes and softmax arrivals land on the even
// CTA's barriers.
template <int HD, bool PAIR>
struct Layout {
    static constexpr int NBOX = HD / 64;
    static constexpr int TILE = kBox * NBOX;            // one 128-row tile of Q (this CTA's rows)
    static constexpr int KTILE = PAIR ? TILE / 2 : TILE;  // this CTA's part of a K tile
    static constexpr int VTILE = PAIR ? TILE / 2 : TILE;  // this CTA's part of a V tile
    static constexpr int KST = 3, VST = PAIR ? 3 : CDSP_VST;  // KST == NSB: K stage n%3 is free once S(n) is
    static constexpr int QST = PAIR ? 2 : 1;  // Q buffers: the next unit's Q lands under this unit's tail
    static constexpr int OFF_Q = 0;
    static constexpr int OFF_K = OFF_Q + QST * TILE;
    static constexpr int OFF_V = OFF_K + KST * KTILE;
    // PAIR: bf16 output staging, 128 rows x 64 columns (128B-swizzled) per softmax group, TMA-stored
    static constexpr int STG = PAIR ? 2 * BM * 128 : 0;
    static constexpr int OFF_STG = OFF_V + VST * VTILE;
    static constexpr int OFF_M = OFF_STG + STG;            // running row max m(n): [NG (tile mod NG)][128] float
    static constexpr int OFF_L = OFF_M + NG * BM * 4;      // epilogue hand-over (m_used, l): [2 unit parity][NG][128] float2
    static constexpr int OFF_QP = OFF_L + 2 * NG * BM * 8;  // query position per row: [2 unit buffer][128] int64
    static constexpr int OFF_BAR = OFF_QP + 2 * BM * 8;
    // Local: u_full[2] (unit buffer published), u_empty[2] (read by every consumer), q_empty[2],
    // s_full[NSB], v_empty[VST], o_full (the last four arrive by MMA commit, multicast to both
    // CTAs of a pair).
    // Leader (the even CTA; the only one in a 1-SM launch): q_full[2], k_full[KST], v_full[VST]
    // (TMA bytes of both CTAs), p_full[NSB], o_free (softmax warps of both CTAs).
    // Pair bookkeeping: c_full[2] (odd CTA: next unit id arrived), c_empty[2] (even CTA: consumed).
    // Epilogue hand-over: l_full[2] (the other softmax groups' row sums are in the unit-parity
    // slot), l_empty[2] (the finishing group has read them).
    // (m(n) goes from one softmax group to the other through named barriers 2, 3.)  Every
    // tcgen05.commit costs the tensor pipe ~30 clk (tools/mma_pattern.cu), so each MMA group
    // commits once: s_full[b] (S(n) done) also frees K stage n % 3 (and, for a unit's last
    // tile, the Q buffer); v_empty[s] (PV(n) done) also tells a rescaling group that O is stable.
    static constexpr int B_UF = 0, B_UE = 2, B_QF = 4, B_QE = 6, B_KF = 8, B_VF = B_KF + KST, B_VE = B_VF + VST,
                         B_SF = B_VE + VST, B_PF = B_SF + NSB, B_OF = B_PF + NSB, B_OE = B_OF + 1, B_CF = B_OE + 1,
                         B_CE = B_CF + 2, B_LF = B_CE + 2, B_LE = B_LF + 2, B_PR = B_LE + 2, NBAR = B_PR + 2;
    static_assert(KST == NSB, "K stages are released through s_full");
    static constexpr int OFF_TMEM_SLOT = OFF_BAR + NBAR * 8;
    static constexpr int OFF_CLAIM = OFF_TMEM_SLOT + 8;     // [2] next unit id (odd CTA of a pair)
    static constexpr int OFF_UNIT = OFF_CLAIM + 8;          // [2] x {unit, n_used}
    // [2][LISTMAX] used KV tiles of the unit in order: tile index | 0x8000 if partial
    static constexpr int LISTMAX = HD == 64 ? kSchedMax : kSchedMax / 2;
    static constexpr int OFF_SCHED = OFF_UNIT + 2 * 16;
    // KV blocks of the launch: segment descriptors [kMaxBlk] and first-tile offsets [kMaxBlk + 1]
    static constexpr int OFF_SEG = OFF_SCHED + 2 * LISTMAX * 2;
    static constexpr int OFF_TOFF = OFF_SEG + kMaxBlk * static_cast<int>(sizeof(cdsp_segments));
    static constexpr int OFF_ROLE = OFF_TOFF + (kMaxBlk + 1) * 4;  // [NG] split-unit role of the finishing group
    static constexpr int SMEM = OFF_ROLE + NG * 4 + 1024;  // + alignment slack
};

constexpr uint32_t COL_O = 0;
__host__ __device__ constexpr uint32_t col_s(int b) { return 128u + 128u * b; }

// A launch walks nblk KV blocks (a ring rank's own store and its peers' stores: P:59 each
// instance "interact[s] local query tensors with full key-value tensors"): every unit's tile
// list runs through block 0, 1, ... in order, with O and the row statistics resident in TMEM /
// registers across blocks, so one launch covers the rank's whole ring.  seg[b] describes
// block b (its query fields are the same in every block); the unit lists use launch-global
// tile ids, block b's tiles being [tile_off[b], tile_off[b + 1]).
struct TcParams {
    cdsp_segments seg[kMaxBlk];
    int tile_off[kMaxBlk + 1];
    int nblk;
    // Arrival gating (ring pulls landing while the launch runs): the first K / V tile of block
    // b (bit b of gate_mask) for KV head kvh is loaded only once
    // gate[b * gate_ng + kvh / gate_hpg] has reached gate_target (written by the stream that
    // pulls the block, behind the pull); a wait longer than ~3 s sets *gate_err and proceeds.
    const uint32_t* gate;
    uint32_t gate_target, gate_mask;
    int gate_ng, gate_hpg;
    int* gate_err;
    int Hq, Hkv, g, n_rb, n_units;
    float scale_log2;
    int mode;
    float* o_acc;
    float* lse_acc;
    __nv_bfloat16* out;
    float* lse;
    int* claim;  // [2]: dynamic unit counter, finished-CTA counter (both zero at launch; the last CTA re-zeroes them)
    int n_pb;    // row blocks per head in units of the CTA group (PAIR: pairs of 128-row blocks)
    // Split units (multi-block launches): the n_split heaviest units of every head (the top row
    // blocks: a unit's work grows with its rows' positions) run as two sub-units, blocks
    // [0, split_blk) and [split_blk, nblk), claimed back to back.  The first
    // to finish writes its normalised partial and LSE into the o_acc / lse_acc rows of the unit
    // (R3 operands), the second merges it with its own and writes the output: a heavy unit no
    // longer sets the launch's tail.  split_cnt: per (unit, CTA) {arrivals, partial-ready}, zero
    // between launches (the second finisher re-zeroes its pair).
    int split, split_blk;  // split: number of split units per head of region B (0: none)
    int n_light, heads_a;  // unit order regions (see unit_map)
    int* split_cnt;
};

// Debug timeline (build with -DCDSP_KTRACE): per-unit phase stamps (globaltimer) and SM id,
// dumped by the host when CDSP_TRACE=<file> is set.
#ifdef CDSP_KTRACE
__device__ unsigned long long g_cta[65536 * 8];  // per unit: published, epi end, smid, used tiles, published, 1st S, loop end, epi end
__device__ __forceinline__ unsigned long long gtime_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ unsigned long long g_it[4 * 512 * 16];  // CTAs 0..3, first 512 tiles, 16 slots
#define KTRACE(slot, iter)                                                                             \
    do {                                                                                               \
        if (blockIdx.x < 4 && (iter) < 512)                                                            \
            g_it[(static_cast<size_t>(blockIdx.x) * 512 + (iter)) * 16 + (slot)] = clock64();          \
    } while (0)
#define UNIT_STAMP(unit, slot, val)                                                              \
    do {                                                                                         \
        if ((unit) < 65536) g_cta[static_cast<size_t>(unit) * 8 + (slot)] = (val);               \
    } while (0)
#else
#define KTRACE(slot, iter) \
    do {                   \
    } while (0)
#define UNIT_STAMP(unit, slot, val) \
    do {                            \
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

__device__ __forceinline__ uint64_t kv_policy() {
#if CDSP_KV_POLICY == 1
    return policy_evict_normal();
#elif CDSP_KV_POLICY == 2
    return policy_evict_first();
#else
    return policy_evict_last();
#endif
}

template <int V>
struct IntC {
    static constexpr int value = V;
};

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

// mask_cols for launch-global tile id gt (block b: tiles [toff[b], toff[b + 1]))
template <int NW>
__device__ __forceinline__ void mask_tile(uint32_t* s, const cdsp_segments* segs, const int* toff, int gt, int64_t qpos,
                                          int col0) {
    int b = 0;
    while (gt >= toff[b + 1]) ++b;
    mask_cols<NW>(s, segs[b], gt - toff[b], qpos, col0);
}

__device__ __forceinline__ float fmax3(float a, float b, float c) {  // FMNMX3 (sm_100)
    float r;
    asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
    return r;
}
__device__ __forceinline__ float max64(const uint32_t* s) {
    // 8 independent chains over 64 scores: 24 FMNMX3 + 8 FMNMX + a 2-level tree
    float a[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = fmax3(__uint_as_float(s[k]), __uint_as_float(s[8 + k]), __uint_as_float(s[16 + k]));
#pragma unroll
    for (int i = 24; i < 56; i += 16)
#pragma unroll
        for (int k = 0; k < 8; ++k) a[k] = fmax3(a[k], __uint_as_float(s[i + k]), __uint_as_float(s[i + 8 + k]));
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = fmaxf(a[k], __uint_as_float(s[56 + k]));
    return fmax3(fmax3(a[0], a[1], a[2]), fmax3(a[3], a[4], a[5]), fmaxf(a[6], a[7]));
}

// lacc += the two bf16 halves of pk, widened exactly (FHADD.BF16: one instruction per half).
__device__ __forceinline__ void add_bf16x2(float2& lacc, uint32_t pk) {
    asm("{\n\t.reg .b16 lo, hi;\n\tmov.b32 {lo, hi}, %2;\n\t"
        "add.rn.f32.bf16 %0, lo, %0;\n\tadd.rn.f32.bf16 %1, hi, %1;\n\t}"
        : "+f"(lacc.x), "+f"(lacc.y)
        : "r"(pk));
}

// p = 2^(s*sl2 - m) for 32 scores -> 16 bf16 pairs stored to TMEM columns tP .. tP+15 (two
// tcgen05.st x8); row sum accumulated in lacc.  Pairs selected by CDSP_EMU_MASK run on the FMA pipe.
// CDSP_SUM_ROUNDED=1 (measured, not the default): the row sum adds the bf16-ROUNDED p the PV
// MMA consumes (FHADD.BF16), so numerator and denominator share their rounding.  Same box:
// 3-7% slower, sharp-q max-abs out 0.021 -> 0.011, but the LSE then carries the bf16 rounding
// of the p (1.3e-3 > the 1e-3 bound); the fp32 sum is kept.
#ifndef CDSP_SUM_ROUNDED
#define CDSP_SUM_ROUNDED 0
#endif
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
#if defined(CDSP_DBG_SOFTMAX) && CDSP_DBG_SOFTMAX == 3
                pp = x;
#else
                pp.x = ex2(x.x);
                pp.y = ex2(x.y);
#endif
            }
            pk[ii] = pack_bf16(pp.x, pp.y);
#if CDSP_SUM_ROUNDED
            add_bf16x2(lacc, pk[ii]);
#else
            lacc = fadd2(lacc, pp);
#endif
        }
#if defined(CDSP_DBG_SOFTMAX) && CDSP_DBG_SOFTMAX == 2
        lacc.x += __uint_as_float(pk[0] ^ pk[1] ^ pk[2] ^ pk[3] ^ pk[4] ^ pk[5] ^ pk[6] ^ pk[7]);
#else
        tmem_st8(tP + 8 * h, pk);
#endif
    }
}

// Work unit x in [0, n_units): head-major (the ~148 units in flight share one head's K/V,
// which stays L2-resident), heavy row blocks first within a head (causal work grows with
// the row).  Units are handed out dynamically (first one = the CTA group's index, then an
// atomic counter), like the hardware's own CTA scheduler but without a CTA's fixed costs
// per unit.  PAIR: a unit is two adjacent 128-row blocks (the even CTA takes the lower).
struct UnitInfo {
    int x, n_used;  // x < 0: no more units
};
constexpr uint16_t kPartialBit = 0x8000;


// Coalesced fp32 row I/O for a warp's 32 rows x 32 columns (row = lane) through a 4 KB
// 128B-swizzled shared-memory tile: global traffic moves 4 whole 128-byte row pieces per warp
// instruction instead of one 16-byte piece of 32 different rows.  base: row 0, first column;
// rows >= nvalid do not exist (read as 0, not written).
__device__ __forceinline__ void warp_rows_load(float (&a)[32], const float* base, size_t rstride, int nvalid,
                                               uint32_t tile, int lane) {
    float4 x[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        const int rr = 4 * k + (lane >> 3), ch = lane & 7;
        x[k] = rr < nvalid ? *reinterpret_cast<const float4*>(base + rr * rstride + ch * 4) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        const int rr = 4 * k + (lane >> 3), ch = lane & 7;
        asm volatile("st.shared.v4.f32 [%0], {%1,%2,%3,%4};" ::"r"(tile + rr * 128 + ((ch ^ (rr & 7)) << 4)),
                     "f"(x[k].x), "f"(x[k].y), "f"(x[k].z), "f"(x[k].w)
                     : "memory");
    }
    __syncwarp();
#pragma unroll
    for (int j = 0; j < 8; ++j)
        asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];"
                     : "=f"(a[4 * j]), "=f"(a[4 * j + 1]), "=f"(a[4 * j + 2]), "=f"(a[4 * j + 3])
                     : "r"(tile + lane * 128 + ((j ^ (lane & 7)) << 4))
                     : "memory");
    __syncwarp();
}
__device__ __forceinline__ void warp_rows_store(const uint32_t* v, float* base, size_t rstride, int nvalid, uint32_t tile,
                                                int lane) {
#pragma unroll
    for (int j = 0; j < 8; ++j)
        asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(tile + lane * 128 + ((j ^ (lane & 7)) << 4)),
                     "r"(v[4 * j]), "r"(v[4 * j + 1]), "r"(v[4 * j + 2]), "r"(v[4 * j + 3])
                     : "memory");
    __syncwarp();
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        const int rr = 4 * k + (lane >> 3), ch = lane & 7;
        float4 x;
        asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];"
                     : "=f"(x.x), "=f"(x.y), "=f"(x.z), "=f"(x.w)
                     : "r"(tile + rr * 128 + ((ch ^ (rr & 7)) << 4))
                     : "memory");
        if (rr < nvalid) *reinterpret_cast<float4*>(base + rr * rstride + ch * 4) = x;
    }
    __syncwarp();
}

// 64 columns (two 32-column chunks, tiles t0 / t1) per round trip: all 16 loads of the warp's
// rows are in flight before the first use.
__device__ __forceinline__ void warp_rows_load64(float (&a)[64], const float* base, size_t rstride, int nvalid,
                                                 uint32_t t0, uint32_t t1, int lane) {
    float4 x[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) {
        const int c = k >> 3, rr = 4 * (k & 7) + (lane >> 3), ch = lane & 7;
        x[k] = rr < nvalid ? *reinterpret_cast<const float4*>(base + rr * rstride + 32 * c + ch * 4)
                           : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int k = 0; k < 16; ++k) {
        const int c = k >> 3, rr = 4 * (k & 7) + (lane >> 3), ch = lane & 7;
        asm volatile("st.shared.v4.f32 [%0], {%1,%2,%3,%4};" ::"r"((c ? t1 : t0) + rr * 128 + ((ch ^ (rr & 7)) << 4)),
                     "f"(x[k].x), "f"(x[k].y), "f"(x[k].z), "f"(x[k].w)
                     : "memory");
    }
    __syncwarp();
#pragma unroll
    for (int j = 0; j < 16; ++j)
        asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];"
                     : "=f"(a[4 * j]), "=f"(a[4 * j + 1]), "=f"(a[4 * j + 2]), "=f"(a[4 * j + 3])
                     : "r"(((j >> 3) ? t1 : t0) + lane * 128 + (((j & 7) ^ (lane & 7)) << 4))
                     : "memory");
    __syncwarp();
}
__device__ __forceinline__ void warp_rows_store64(const uint32_t* v, float* base, size_t rstride, int nvalid,
                                                  uint32_t t0, uint32_t t1, int lane) {
#pragma unroll
    for (int j = 0; j < 16; ++j)
        asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(((j >> 3) ? t1 : t0) + lane * 128 +
                                                                     (((j & 7) ^ (lane & 7)) << 4)),
                     "r"(v[4 * j]), "r"(v[4 * j + 1]), "r"(v[4 * j + 2]), "r"(v[4 * j + 3])
                     : "memory");
    __syncwarp();
#pragma unroll
    for (int k = 0; k < 16; ++k) {
        const int c = k >> 3, rr = 4 * (k & 7) + (lane >> 3), ch = lane & 7;
        float4 x;
        asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];"
                     : "=f"(x.x), "=f"(x.y), "=f"(x.z), "=f"(x.w)
                     : "r"((c ? t1 : t0) + rr * 128 + ((ch ^ (rr & 7)) << 4))
                     : "memory");
        if (rr < nvalid) *reinterpret_cast<float4*>(base + rr * rstride + 32 * c + ch * 4) = x;
    }
    __syncwarp();
}

// TMA descriptors: queries, bf16 output, and K / V of every block (kernel-parameter space)
struct TcMaps {
    CUtensorMap q, out;
    CUtensorMap k[kMaxBlk], v[kMaxBlk];
};

// Block b of the unit's KV walk has arrived: spin (acquire, system scope: the block is written
// by copy engines, possibly of a peer GPU) until the gate word reaches the target, then order
// the async proxy (TMA) after it.
__device__ __forceinline__ void gate_wait(const TcParams& p, int b, int kvh) {
    const uint32_t* f = p.gate + b * p.gate_ng + kvh / p.gate_hpg;
    const uint64_t t0 = globaltimer();
    for (;;) {
        uint32_t v;
        asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
        if (static_cast<int32_t>(v - p.gate_target) >= 0) break;
        if (globaltimer() - t0 > 3000000000ull) {  // before the 4 s mbarrier watchdogs of the other warps
            atomicExch(p.gate_err, 3);
            break;
        }
        __nanosleep(128);
    }
    asm volatile("fence.proxy.async.global;" ::: "memory");
}

// Role of a finishing group in a split unit's pair protocol (all BM threads of group g call it):
// 1 = first (leave the partial in the accumulator rows), 0 = second (wait for the partner's
// partial, re-zero the pair's counters).  Out of line: its registers stay out of the softmax.
__device__ __noinline__ int split_role(int* scnt, volatile int* role, int bar_id, int nthreads, bool leader) {
    if (leader) *role = atomicAdd(scnt, 1);
    named_bar_sync(bar_id, nthreads);
    const int first = *role == 0;
    if (!first) {
        if (leader) {  // the partner is past its own atomicAdd: it is writing its partial
            const uint64_t t0 = globaltimer();
            for (;;) {
                int f;
                asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(f) : "l"(scnt + 1) : "memory");
                if (f != 0) break;
                if (globaltimer() - t0 > 3000000000ull) __trap();
                __nanosleep(64);
            }
            scnt[0] = 0;  // both parties are done with the pair: zero for the next launch
            scnt[1] = 0;
        }
        named_bar_sync(bar_id, nthreads);
        __threadfence();
    }
    return first;
}

template <int HD, bool PAIR>
__global__ void __maxnreg__(CDSP_REGSPLIT ? 128 : CDSP_MAXNREG)
    attn_tc_kernel(const __grid_constant__ TcMaps tm, const __grid_constant__ TcParams p) {
    using L = Layout<HD, PAIR>;
    extern __shared__ uint8_t smem_raw[];
    // 1024-byte alignment for the 128B-swizzle atoms
    const uint32_t raw_addr = smem_u32(smem_raw);
    uint8_t* smem = smem_raw + ((1024u - (raw_addr & 1023u)) & 1023u);
    const uint32_t sbase = smem_u32(smem);
    const uint32_t sQ = sbase + L::OFF_Q, sK = sbase + L::OFF_K, sV = sbase + L::OFF_V;
    const uint32_t bar0 = sbase + L::OFF_BAR;
    auto bar = [&](int i) { return bar0 + 8u * static_cast<uint32_t>(i); };
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + L::OFF_TMEM_SLOT);
    UnitInfo* uinfo = reinterpret_cast<UnitInfo*>(smem + L::OFF_UNIT);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const cdsp_segments* segs = reinterpret_cast<const cdsp_segments*>(smem + L::OFF_SEG);
    const int* toff = reinterpret_cast<const int*>(smem + L::OFF_TOFF);
    const cdsp_segments& sg = segs[0];  // query fields (the same in every block)
    constexpr int CL = PAIR ? 2 : 1;
    const int crank = PAIR ? static_cast<int>(cluster_ctarank()) : 0;
    const bool leader = crank == 0;
    const int G = static_cast<int>(gridDim.x) / CL;  // CTA groups
    // the leader's barrier i as seen from this CTA (TMA bytes / arrivals of both CTAs land there)
    auto lbar = [&](int i) { return PAIR ? mapa_shared(bar(i), 0) : bar(i); };
    // unit x -> head, first row, part (-1: whole unit; 0 / 1: sub-unit of a split unit whose
    // counter index is *ux) and its block range [*b0, *b1)
    // Order (three regions):
    //  A  heads [0, heads_a): the heavy row blocks (pb >= n_light) head-major, heaviest first
    //     within a head — the units in flight share a few heads' K/V in L2 (every unit of a head
    //     streams the same tiles);
    //  B  heads [heads_a, Hq): the same, the n_split heaviest units of each head as two adjacent
    //     sub-units (the launch's last wave comes in halves: no heavy unit sets the tail);
    //  C  every head's light row blocks (pb < n_light), which fill the tail.
    auto unit_map = [&](int x, int c, int& head, int64_t& row0, int& part, int& ux, int& b0, int& b1) {
        int pb;
        part = -1;
        b0 = 0;
        b1 = p.nblk;
        ux = x;
        const int nh = p.n_pb - p.n_light;       // heavy row blocks per head
        const int na = p.heads_a * nh;           // region A units
        const int nbh = nh + p.split;            // region B units per head
        const int nb = (p.Hq - p.heads_a) * nbh;
        if (x < na) {
            head = x / nh;
            pb = p.n_pb - 1 - (x - head * nh);
        } else if (x < na + nb) {
            const int xb = x - na;
            const int hb = xb / nbh, y = xb - hb * nbh;
            head = p.heads_a + hb;
            if (y < 2 * p.split) {
                part = y & 1;
                pb = p.n_pb - 1 - (y >> 1);
                ux = hb * p.split + (y >> 1);
                if (part == 0) b1 = p.split_blk;
                else b0 = p.split_blk;
            } else {
                pb = p.n_pb - 1 - (y - p.split);
            }
        } else {
            const int xc = x - na - nb;
            head = xc / p.n_light;
            pb = p.n_light - 1 - (xc - head * p.n_light);
        }
        row0 = static_cast<int64_t>(PAIR ? 2 * pb + c : pb) * BM;
    };
    auto unit_rows = [&](int x, int c, int& head, int64_t& row0) {
        int part, ux, b0, b1;
        unit_map(x, c, head, row0, part, ux, b0, b1);
    };

    // ---- unit epilogue (one group's finish of a unit): normalise O, then write the bf16 output
    // or the fp32 accumulator / LSE-merge with it (R3).  Instantiated per role (MG: merge with
    // the accumulator, TA: write to it; 0 / 1 fixed, 2 the launch's mode).  Columns [64 hh0,
    // 64 hh1) of O; wide_ok: 64-column accumulator round trips through this group's 8 KB per
    // warp of staging; write_lse: this group writes the row's LSE.
    const int64_t nq = p.seg[0].nq;  // (the shared-memory copy sg is written in setup, below)
    const bool l_merge = p.mode == CDSP_ATTN_MID || p.mode == CDSP_ATTN_LAST;
    const bool l_to_acc = p.mode == CDSP_ATTN_FIRST || p.mode == CDSP_ATTN_MID;
    auto arrive_leader = [&](int b) {  // lane 0, after the warp's tcgen05 ops are fenced
        if constexpr (PAIR) mbar_arrive_remote(lbar(b));
        else mbar_arrive(bar(b));
    };
    auto run_epilogue = [&](auto MG, auto TA, const int head, const int64_t row0, const int64_t row, const bool row_ok,
                            const int r, const int quad, const int N, const float l, const float m,
                            const int n_units_done, const uint32_t tO, const int stage_bar, const unsigned stage_lead,
                            const int hh0, const int hh1, const bool wide_ok, const bool write_lse) {
        const bool merge = decltype(MG)::value == 2 ? l_merge : decltype(MG)::value == 1;
        const bool to_acc = decltype(TA)::value == 2 ? l_to_acc : decltype(TA)::value == 1;
        const float lse_a = merge && row_ok ? p.lse_acc[static_cast<size_t>(head) * nq + row] : -INFINITY;
        const float inv_l = l > 0.f ? 1.0f / l : 0.f;
        const float lse_b = l > 0.f ? (m + __log2f(l)) * 0.69314718055994530942f : -INFINITY;
        float wa = 0.f, wb = 1.f, lse_out = lse_b;
        if (merge) merge_weights(lse_a, lse_b, wa, wb, lse_out);
        const float sbw = wb * inv_l;
        // PAIR: bf16 rows go through two 128B-swizzled boxes (64 columns each) and TMA stores;
        // fp32 accumulator rows through each warp's 4 KB slices of the same boxes (coalesced)
        const bool boxed = PAIR && N > 0 && (CDSP_EPI_COALESCED || !to_acc);
        const uint32_t stg0 = sbase + L::OFF_STG;
        const int64_t wrow0 = row0 + 32 * quad;
        const int nvalid = static_cast<int>(nq - wrow0 < 32 ? (nq - wrow0 > 0 ? nq - wrow0 : 0) : 32);
        const size_t rstride = static_cast<size_t>(p.Hq) * HD;
#pragma unroll 1
        for (int hh = hh0; hh < hh1; ++hh) {  // O columns [64 hh, 64 hh + 64)
            uint32_t o[64];
            if (N > 0) {
                if (hh == hh0) {
                    mbar_wait(bar(L::B_OF), (n_units_done - 1) & 1);
                    tc_fence_after();
                }
                tmem_ld32p(tO + 64 * hh, o);
                tmem_ld32p(tO + 64 * hh + 32, o + 32);
                tc_wait_ld();
                reg_tie32(o);
                reg_tie32(o + 32);
                if (hh == hh1 - 1) {  // O drained: TMEM back to the next unit's PV
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) arrive_leader(L::B_OE);
                }
            } else {
#pragma unroll
                for (int q = 0; q < 64; ++q) o[q] = 0u;
            }
            if (boxed && to_acc && CDSP_EPI_WIDE && wide_ok) {
                // fp32 accumulator, FIRST / MID: the finishing group alone uses the 32 KB of
                // boxes, so this warp's 8 KB (its rows of both boxes) carry a 64-column half
                // per round trip
                const uint32_t t0 = stg0 + static_cast<uint32_t>(quad) * (32 * 128);
                const uint32_t t1 = t0 + BM * 128;
                float* acc_w = p.o_acc + (static_cast<size_t>(nvalid > 0 ? wrow0 : 0) * p.Hq + head) * HD + 64 * hh;
                if (merge) {
                    float a[64];
                    warp_rows_load64(a, acc_w, rstride, nvalid, t0, t1, lane);
#pragma unroll
                    for (int q = 0; q < 64; ++q) o[q] = __float_as_uint(fmaf(wa, a[q], __uint_as_float(o[q]) * sbw));
                } else {
#pragma unroll
                    for (int q = 0; q < 64; ++q) o[q] = __float_as_uint(__uint_as_float(o[q]) * sbw);
                }
                warp_rows_store64(o, acc_w, rstride, nvalid, t0, t1, lane);
            } else if (boxed) {
                const uint32_t box = stg0 + static_cast<uint32_t>(hh) * (BM * 128);
                const uint32_t wtile = box + static_cast<uint32_t>(quad) * (32 * 128);
                float* acc_w = p.o_acc + (static_cast<size_t>(nvalid > 0 ? wrow0 : 0) * p.Hq + head) * HD + 64 * hh;
#pragma unroll
                for (int c = 0; c < 2; ++c) {
                    float a[32];
                    if (merge) warp_rows_load(a, acc_w + 32 * c, rstride, nvalid, wtile, lane);
#pragma unroll
                    for (int q = 0; q < 32; ++q) {
                        float v = __uint_as_float(o[32 * c + q]) * sbw;
                        if (merge) v = fmaf(wa, a[q], v);
                        o[32 * c + q] = __float_as_uint(v);
                    }
                }
                if (to_acc) {
#pragma unroll
                    for (int c = 0; c < 2; ++c) warp_rows_store(o + 32 * c, acc_w + 32 * c, rstride, nvalid, wtile, lane);
                } else {
                    const uint32_t rsw = static_cast<uint32_t>(r & 7), rowa = box + static_cast<uint32_t>(r) * 128;
#pragma unroll
                    for (int q = 0; q < 8; ++q) {  // 16-byte chunk q of the 128-byte row
                        const uint32_t* w = o + 8 * q;
                        asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(rowa + ((static_cast<uint32_t>(q) ^ rsw) << 4)),
                                     "r"(pack_bf16(__uint_as_float(w[0]), __uint_as_float(w[1]))),
                                     "r"(pack_bf16(__uint_as_float(w[2]), __uint_as_float(w[3]))),
                                     "r"(pack_bf16(__uint_as_float(w[4]), __uint_as_float(w[5]))),
                                     "r"(pack_bf16(__uint_as_float(w[6]), __uint_as_float(w[7])))
                                     : "memory");
                    }
                }
            } else if (row_ok) {
                const size_t orow = (static_cast<size_t>(row) * p.Hq + head) * HD + 64 * hh;
#pragma unroll
                for (int c = 0; c < 2; ++c) {
                    float v[32];
#pragma unroll
                    for (int q = 0; q < 32; ++q) v[q] = __uint_as_float(o[32 * c + q]) * sbw;
                    if (merge) {
                        const float4* a4 = reinterpret_cast<const float4*>(p.o_acc + orow + 32 * c);
#pragma unroll
                        for (int q = 0; q < 8; ++q) {
                            const float4 av = a4[q];
                            v[4 * q + 0] = fmaf(wa, av.x, v[4 * q + 0]);
                            v[4 * q + 1] = fmaf(wa, av.y, v[4 * q + 1]);
                            v[4 * q + 2] = fmaf(wa, av.z, v[4 * q + 2]);
                            v[4 * q + 3] = fmaf(wa, av.w, v[4 * q + 3]);
                        }
                    }
                    if (to_acc) {
                        float4* d4 = reinterpret_cast<float4*>(p.o_acc + orow + 32 * c);
#pragma unroll
                        for (int q = 0; q < 8; ++q) d4[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
                    } else {
                        uint4* d4 = reinterpret_cast<uint4*>(p.out + orow + 32 * c);
#pragma unroll
                        for (int q = 0; q < 4; ++q)
                            d4[q] = make_uint4(pack_bf16(v[8 * q + 0], v[8 * q + 1]), pack_bf16(v[8 * q + 2], v[8 * q + 3]),
                                               pack_bf16(v[8 * q + 4], v[8 * q + 5]), pack_bf16(v[8 * q + 6], v[8 * q + 7]));
                    }
                }
            }
        }
        if (boxed && !to_acc) {
            fence_proxy_async_smem();
            named_bar_sync(stage_bar, BM);  // this group's 128 rows are in the boxes
            if (threadIdx.x == stage_lead) {
                for (int hh = hh0; hh < hh1; ++hh)
                    tma_store_3d(&tm.out, stg0 + static_cast<uint32_t>(hh) * (BM * 128), 64 * hh, head,
                                 static_cast<int>(row0));  // rows >= nq clipped
                bulk_commit();
                // the boxes are free again once the engine has read them: at once when both
                // softmax groups share them, else before this group's next use (epilogue group)
                if (!CDSP_EPI_WARPS) bulk_wait_read0();
            }
        }
        if (row_ok && write_lse) {
            const size_t li = static_cast<size_t>(head) * nq + row;
            if (to_acc) {
                p.lse_acc[li] = lse_out;
            } else if (p.lse) {
                p.lse[li] = lse_out;
            }
        }
    };

    // ---- setup (once per CTA)
    if (warp == W_K) {
        if (lane == 0) {
            for (int i = 0; i < 2; ++i) {
                mbar_init(bar(L::B_UF + i), ARRIVERS);  // the scheduler warp (its list / position writes)
                mbar_init(bar(L::B_UE + i), ARRIVERS * (4 * NG + NEPI + 3));  // softmax, epilogue, K / V producers, MMA warps
                mbar_init(bar(L::B_CF + i), 1);
                mbar_init(bar(L::B_CE + i), 1);
            }
            for (int i = 0; i < 2; ++i) {
                mbar_init(bar(L::B_QF + i), 1);
                mbar_init(bar(L::B_QE + i), 1);
            }
            for (int i = 0; i < L::KST; ++i) mbar_init(bar(L::B_KF + i), 1);
            for (int i = 0; i < L::VST; ++i) {
                mbar_init(bar(L::B_VF + i), 1);
                mbar_init(bar(L::B_VE + i), 1);
            }
            for (int b = 0; b < NSB; ++b) {
                mbar_init(bar(L::B_SF + b), 1);
                mbar_init(bar(L::B_PF + b), 4 * CL);  // the softmax warps of the tile (x CTAs of a pair)
            }
            mbar_init(bar(L::B_OF), 1);
            mbar_init(bar(L::B_OE), 4 * CL);  // the finishing group's 4 warps (x CTAs of a pair)
            for (int i = 0; i < 2; ++i) {
                // row statistics hand-over: every softmax group to the epilogue group (CDSP_EPI_WARPS),
                // else the other groups to the finishing one
                mbar_init(bar(L::B_LF + i), ARRIVERS * 4 * (CDSP_EPI_WARPS ? NG : NG - 1));
                mbar_init(bar(L::B_LE + i), ARRIVERS * 4);
                mbar_init(bar(L::B_PR + i), 1);  // the K producer is kPrepLead tiles from the unit's end
            }
            fence_barrier_init();
            tma_prefetch_desc(&tm.q);
            for (int b = 0; b < p.nblk; ++b) {
                tma_prefetch_desc(&tm.k[b]);
                tma_prefetch_desc(&tm.v[b]);
            }
            if (PAIR) tma_prefetch_desc(&tm.out);
        }
        // block table into shared memory (read by the producers and on partial tiles)
        const int64_t* src = reinterpret_cast<const int64_t*>(p.seg);
        int64_t* dst = reinterpret_cast<int64_t*>(smem + L::OFF_SEG);
        constexpr int nw = kMaxBlk * static_cast<int>(sizeof(cdsp_segments)) / 8;
        for (int i = lane; i < nw; i += 32) dst[i] = src[i];
        for (int i = lane; i <= kMaxBlk; i += 32) reinterpret_cast<int*>(smem + L::OFF_TOFF)[i] = p.tile_off[i];
    } else if (warp == W_MMA) {
        if constexpr (PAIR) {
            tmem_alloc2(smem_u32(tmem_slot), 512);
            tmem_relinquish2();
        } else {
            tmem_alloc(smem_u32(tmem_slot), 512);
            tmem_relinquish();
        }
    }
    tc_fence_before();
    if constexpr (PAIR) cluster_sync_all();  // both CTAs' barriers exist before any remote arrive
    else __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

#if CDSP_REGSPLIT
    if (warp >= W_K) asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(CDSP_PRODUCER_REGS) : "memory");  // producers, MMA issuer
#endif
    if (warp == W_SCH) {
        // ======== unit scheduler: claim each unit, list its used KV tiles in order (empty ones
        // skipped), publish it (u_full[i&1]; its slot is free once every consumer, the K producer
        // included, is done with the unit two back) and load its Q tile once the Q buffer is
        // free.  Its own warp: list building and the claim round trip stay off the K stream ========
        const uint64_t pol_q = policy_evict_first();
        int x = static_cast<int>(blockIdx.x) / CL;
        int x_pre = 0;  // leader lane 0: the unit after x, claimed one unit ahead
        if (leader && lane == 0) x_pre = G + atomicAdd(p.claim, 1);
        int n_ne = 0;      // non-empty units so far
        int* claim_slot = reinterpret_cast<int*>(smem + L::OFF_CLAIM);
        // prepare unit i (its id in x): list, publish, Q; returns its tile count (-1: no more units)
        auto prepare = [&](int i) -> int {
            const int ub = i & 1;
            if (i >= 1) {  // unit id: the even CTA claims one unit ahead and tells the odd CTA
                x = __shfl_sync(0xFFFFFFFFu, x_pre, 0);
                if (leader && lane == 0) {
                    if (x < p.n_units) x_pre = G + atomicAdd(p.claim, 1);
                    if constexpr (PAIR) {  // message i to the odd CTA: the unit it runs next
                        const int s = (i - 1) & 1, use = (i - 1) >> 1;
                        if (use >= 1) mbar_wait(bar(L::B_CE + s), (use - 1) & 1);  // slot consumed
                        st_cluster_u32(mapa_shared(smem_u32(claim_slot + s), 1), static_cast<uint32_t>(x));
                        mbar_arrive_cluster(mapa_shared(bar(L::B_CF + s), 1));
                    }
                }
                __syncwarp();
                if constexpr (PAIR) {
                    if (!leader) {  // unit id from the even CTA (message i)
                        const int s = (i - 1) & 1, use = (i - 1) >> 1;
                        mbar_wait_acq_cluster(bar(L::B_CF + s), use & 1);  // pairs with the even CTA's release.cluster
                        x = *reinterpret_cast<volatile int*>(claim_slot + s);
                        __syncwarp();
                        if (lane == 0) mbar_arrive_remote(mapa_shared(bar(L::B_CE + s), 0));
                    }
                }
            }
            if (i >= 2) mbar_wait(bar(L::B_UE + ub), ((i - 2) >> 1) & 1);  // every consumer is done with unit i-2
            if (x >= p.n_units) {
                if (lane == 0) uinfo[ub].x = -1;
                __syncwarp();
                if (ARRIVE_LANE) mbar_arrive(bar(L::B_UF + ub));
                // no more units here: a programmatically dependent launch (the next ring step)
                // may start on the SMs this grid frees from now on
                if (lane == 0) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
                return -1;
            }
            int head, part, ux, blo, bhi;
            int64_t row0;
            unit_map(x, crank, head, row0, part, ux, blo, bhi);
            uint16_t* list = reinterpret_cast<uint16_t*>(smem + L::OFF_SCHED) + ub * L::LISTMAX;
            int64_t qlo, qhi, plo = 0, phi = 0;
            bool qany, pany = false;
            seg_qrange(sg, row0, row0 + BM, qlo, qhi, qany);
            if constexpr (PAIR) {  // the peer's rows: the pair walks the union of both schedules
                int ph;
                int64_t prow0;
                unit_rows(x, 1 - crank, ph, prow0);
                seg_qrange(sg, prow0, prow0 + BM, plo, phi, pany);
            }
            int cnt = 0;
            for (int b = blo; b < bhi; ++b) {  // blocks in walk order, each block's tiles in order
                const cdsp_segments& sb = segs[b];
                const int t0 = toff[b], nt = toff[b + 1] - t0;
                for (int j0 = 0; j0 < nt; j0 += 32) {  // 32 tiles per step, compacted in order
                    const int j = j0 + lane;
                    int k = TILE_EMPTY;
                    if (j < nt) {
                        k = seg_tile_kind(sb, qany, qlo, qhi, static_cast<int64_t>(j) * BN, BN);
                        if (PAIR && k == TILE_EMPTY &&
                            seg_tile_kind(sb, pany, plo, phi, static_cast<int64_t>(j) * BN, BN) != TILE_EMPTY)
                            k = TILE_PARTIAL;  // needed by the peer only: fully masked here
                    }
                    const uint32_t used = __ballot_sync(0xFFFFFFFFu, k != TILE_EMPTY);
                    if (k != TILE_EMPTY)
                        list[cnt + __popc(used & ((1u << lane) - 1u))] =
                            static_cast<uint16_t>((t0 + j) | (k == TILE_PARTIAL ? kPartialBit : 0));
                    cnt += __popc(used);
                }
            }
            // query positions (only read on partial tiles)
            int64_t* qp = reinterpret_cast<int64_t*>(smem + L::OFF_QP) + ub * BM;
            for (int rr = lane; rr < BM; rr += 32) {
                const int64_t row = row0 + rr;
                qp[rr] = row < sg.nq ? seg_qpos(sg, row) : (INT64_MAX >> 2);
            }
            if (lane == 0) uinfo[ub] = UnitInfo{x, cnt};
            __threadfence_block();
            __syncwarp();
            if (ARRIVE_LANE) mbar_arrive(bar(L::B_UF + ub));  // publish (release)
            if (cnt > 0) {
                // Q buffer qb is free once the last S of the unit that used it (n_ne - QST) is done
                const int qb = n_ne % L::QST;
                if (n_ne >= L::QST) mbar_wait(bar(L::B_QE + qb), ((n_ne - L::QST) / L::QST) & 1);
                if (lane == 0) {
                    UNIT_STAMP(x * CL + crank, 0, gtime_ns());
                    if (leader) mbar_expect_tx(bar(L::B_QF + qb), CL * L::TILE);
                    const uint32_t dst = sQ + qb * L::TILE;
                    for (int b = 0; b < L::NBOX; ++b) {
                        if constexpr (PAIR)
                            tma_load_3d_2sm(dst + b * kBox, &tm.q, lbar(L::B_QF + qb), b * 64, head, static_cast<int>(row0),
                                            pol_q);
                        else
                            tma_load_3d(dst + b * kBox, &tm.q, bar(L::B_QF + qb), b * 64, head, static_cast<int>(row0));
                    }
                }
                // merge modes: pull this unit's accumulator rows into L2 for the epilogue
                if ((p.mode == CDSP_ATTN_MID || p.mode == CDSP_ATTN_LAST) && part < 0) {
                    for (int rr = lane; rr < BM; rr += 32) {
                        const int64_t row = row0 + rr;
                        if (row < sg.nq) {
                            const float* src = p.o_acc + (static_cast<size_t>(row) * p.Hq + head) * HD;
                            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(HD * 4) : "memory");
                        }
                    }
                }
                ++n_ne;
            }
            __syncwarp();
            return cnt;
        };
        // unit i is claimed and prepared once the K producer is kPrepLead tiles from the end of
        // unit i - 1: late enough that the claim order still balances the launch's tail, early
        // enough that the list, the publication and the Q load are done when its first S is due
        for (int i = 0;; ++i) {
            if (i >= 1) mbar_wait(bar(L::B_PR + ((i - 1) & 1)), ((i - 1) >> 1) & 1);
            if (prepare(i) < 0) break;
        }
    } else if (warp == W_K) {
        // ======== TMA producer of K (3 stages), following the published units ========
        const uint64_t pol_kv = kv_policy();
        int it = 0;
        for (int i = 0;; ++i) {
            const int ub = i & 1;
            mbar_wait(bar(L::B_UF + ub), (i >> 1) & 1);
            const UnitInfo u = uinfo[ub];
            if (u.x < 0) break;
            int head;
            int64_t row0_unused;
            unit_rows(u.x, crank, head, row0_unused);
            const int kvh = head / p.g;
            const int cnt = u.n_used;
            const uint16_t* list = reinterpret_cast<const uint16_t*>(smem + L::OFF_SCHED) + ub * L::LISTMAX;
            const int n_prep = cnt > kPrepLead ? cnt - kPrepLead : 0;  // the scheduler's cue for the next unit
            if (n_prep == 0 && lane == 0) mbar_arrive(bar(L::B_PR + ub));
            int blk = 0;  // block of the current list entry (the list runs through blocks in order)
            uint32_t gated = 0;  // gated blocks already seen arrived (this unit)
            for (int n = 0; n < cnt; ++n) {
                if (n == n_prep && n > 0 && lane == 0) mbar_arrive(bar(L::B_PR + ub));
                const int gt = list[n] & ~kPartialBit;
                while (gt >= toff[blk + 1]) ++blk;
                const int j = gt - toff[blk];
                if (((p.gate_mask & ~gated) >> blk) & 1u) {
                    if (lane == 0) gate_wait(p, blk, kvh);
                    __syncwarp();
                    gated |= 1u << blk;
                }
                const int st = it % L::KST;
                // stage st last held tile it - 3: free once S(it - 3) is done (in both CTAs)
                if (it >= L::KST) mbar_wait_backoff(bar(L::B_SF + st), ((it - L::KST) / L::KST) & 1);
                if (lane == 0) KTRACE(15, it);
                if (CDSP_DBG_NO_KV & 1) {  // debug probe: no K traffic (results garbage)
                    if (leader && lane == 0) mbar_arrive(bar(L::B_KF + st));
                } else if (elect_one()) {
                    if constexpr (PAIR) {
                        // this CTA's 64 keys of the tile, both d halves
                        if (leader) mbar_expect_tx(bar(L::B_KF + st), 2 * L::KTILE);
                        for (int b = 0; b < L::NBOX; ++b)
                            tma_load_3d_2sm(sK + st * L::KTILE + b * (kBox / 2), &tm.k[blk], lbar(L::B_KF + st), b * 64,
                                            kvh, j * BN + crank * (BN / 2), pol_kv);
                    } else {
                        mbar_expect_tx(bar(L::B_KF + st), L::KTILE);
                        for (int b = 0; b < L::NBOX; ++b)
                            tma_load_3d_hint(sK + st * L::KTILE + b * kBox, &tm.k[blk], bar(L::B_KF + st), b * 64, kvh,
                                             j * BN, pol_kv);
                    }
                }
                __syncwarp();
                ++it;
            }
            __syncwarp();
            if (ARRIVE_LANE) mbar_arrive(bar(L::B_UE + ub));  // done with the unit's list
        }
    } else if (warp == W_V) {
        // ======== TMA producer of V, following the published units ========
        const uint64_t pol_kv = kv_policy();
        int it = 0;
        for (int i = 0;; ++i) {
            const int ub = i & 1;
            mbar_wait(bar(L::B_UF + ub), (i >> 1) & 1);
            const UnitInfo u = uinfo[ub];
            if (u.x < 0) break;
            int head;
            int64_t row0_unused;
            unit_rows(u.x, crank, head, row0_unused);
            const int kvh = head / p.g;
            const uint16_t* list = reinterpret_cast<const uint16_t*>(smem + L::OFF_SCHED) + ub * L::LISTMAX;
            int blk = 0;
            uint32_t gated = 0;
            for (int n = 0; n < u.n_used; ++n) {
                const int gt = list[n] & ~kPartialBit;
                while (gt >= toff[blk + 1]) ++blk;
                const int j = gt - toff[blk];
                if (((p.gate_mask & ~gated) >> blk) & 1u) {
                    if (lane == 0) gate_wait(p, blk, kvh);
                    __syncwarp();
                    gated |= 1u << blk;
                }
                const int st = it % L::VST;
                if (it >= L::VST) mbar_wait_backoff(bar(L::B_VE + st), ((it - L::VST) / L::VST) & 1);
                if (lane == 0) KTRACE(14, it);
                if (CDSP_DBG_NO_KV & 2) {  // debug probe: no V traffic (results garbage)
                    if (leader && lane == 0) mbar_arrive(bar(L::B_VF + st));
                } else if (elect_one()) {
                    if constexpr (PAIR) {  // all 128 keys, this CTA's 64 d columns
                        if (leader) mbar_expect_tx(bar(L::B_VF + st), 2 * L::VTILE);
                        tma_load_3d_2sm(sV + st * L::VTILE, &tm.v[blk], lbar(L::B_VF + st), crank * 64, kvh, j * BN,
                                        pol_kv);
                    } else {
                        mbar_expect_tx(bar(L::B_VF + st), L::VTILE);
                        for (int b = 0; b < L::NBOX; ++b)
                            tma_load_3d_hint(sV + st * L::VTILE + b * kBox, &tm.v[blk], bar(L::B_VF + st), b * 64, kvh,
                                             j * BN, pol_kv);
                    }
                }
                __syncwarp();
                ++it;
            }
            __syncwarp();
            if (ARRIVE_LANE) mbar_arrive(bar(L::B_UE + ub));
        }
    } else if (warp == W_MMA) {
        // ================= MMA issuer (warp-uniform loop, one lane issues; PAIR: the even CTA) =================
        constexpr uint32_t idesc_qk = idesc_bf16_f32(BM * CL, BN, false, false);
        constexpr uint32_t idesc_pv = idesc_bf16_f32(BM * CL, HD, false, true);
        constexpr uint32_t KBOX = PAIR ? kBox / 2 : kBox;  // bytes of one 64-column box of a K stage
        const uint64_t dq0 = umma_desc_sw128(sQ, 16, 1024);
        uint64_t dq = dq0;
        const uint64_t dk0 = umma_desc_sw128(sK, 16, 1024);
        const uint64_t dv0 = umma_desc_sw128(sV, kBox, 1024);
        auto commit = [&](int b) {
            if constexpr (PAIR) mma_commit2_mc(bar(b), 0x3);
            else mma_commit(bar(b));
        };
        // S(b) = Q K^T: M=128 (x2), N=128, K=HD in steps of 16 (32 B inside a 128-B swizzle row)
        auto issue_qk = [&](int ks, int b, uint64_t dq) {
            const uint64_t dk = dk0 + static_cast<uint64_t>((ks * L::KTILE) >> 4);
#pragma unroll
            for (int kk = 0; kk < HD / 16; ++kk) {
                const uint64_t offq = static_cast<uint64_t>(((kk / 4) * kBox + (kk % 4) * 32) >> 4);
                const uint64_t offk = static_cast<uint64_t>(((kk / 4) * KBOX + (kk % 4) * 32) >> 4);
                if constexpr (PAIR) mma_ss2(tmem + col_s(b), dq + offq, dk + offk, idesc_qk, kk > 0 ? 1u : 0u);
                else mma_ss(tmem + col_s(b), dq + offq, dk + offk, idesc_qk, kk > 0 ? 1u : 0u);
            }
        };
        // O += P(b) V: M=128 (x2), N=HD, K=128 keys in steps of 16 (V rows, 2048 B); P(b) is bf16
        // in the S(b) columns (8 TMEM columns per 16 keys)
        auto issue_pv = [&](int vs, int b, bool acc) {
            const uint64_t dv = dv0 + static_cast<uint64_t>((vs * L::VTILE) >> 4);
#pragma unroll
            for (int kk = 0; kk < BN / 16; ++kk) {
                if constexpr (PAIR)
                    mma_ts2(tmem + COL_O, tmem + col_s(b) + kk * 8, dv + static_cast<uint64_t>((kk * 16 * 128) >> 4),
                            idesc_pv, (acc || kk > 0) ? 1u : 0u);
                else
                    mma_ts(tmem + COL_O, tmem + col_s(b) + kk * 8, dv + static_cast<uint64_t>((kk * 16 * 128) >> 4),
                           idesc_pv, (acc || kk > 0) ? 1u : 0u);
            }
        };
        // S(gn) into buffer gn % NSB; K stage gn % KST; Q of the tile's unit at dq_u
        auto issue_s = [&](int gn, int q_release, uint64_t dq_u) {
            const int ks = gn % L::KST;
            MMA_WAIT(bar(L::B_KF + ks), (gn / L::KST) & 1);
            tc_fence_after();
            if (elect_one()) {
                KTRACE(9, gn);
                issue_qk(ks, gn % NSB, dq_u);
                commit(L::B_SF + gn % NSB);  // S(gn) ready; K stage ks free
                if (q_release >= 0) commit(L::B_QE + q_release);  // the unit's last S: Q buffer free
            }
            __syncwarp();
        };
        auto wait_softmax = [&](int b, uint32_t parity) { MMA_WAIT(bar(b), parity); };
        int gn0 = 0, n_units_done = 0;
        for (int i = 0;; ++i) {
            const int ub = i & 1;
            MMA_WAIT(bar(L::B_UF + ub), (i >> 1) & 1);  // unit published
            const UnitInfo u = uinfo[ub];
            __syncwarp();
            if (ARRIVE_LANE) mbar_arrive(bar(L::B_UE + ub));
            if (u.x < 0) break;
            const int N = u.n_used;
            if (N == 0 || !leader) continue;
            const int qb = n_units_done % L::QST;
            MMA_WAIT(bar(L::B_QF + qb), (n_units_done / L::QST) & 1);  // Q tile(s) landed
            tc_fence_after();
            dq = dq0 + static_cast<uint64_t>((qb * L::TILE) >> 4);
            // this unit's first S tiles go in only after the previous unit's last PV (their buffers
            // are the ones those PVs read).  Issuing each as soon as its buffer's PV is issued, i.e.
            // between the previous unit's last PVs, was measured slower (DESIGN 6.1): that unit's O
            // then completes later and its finishing group reaches its next tile later.
            for (int n = 0; n < NSB && n < N; ++n) issue_s(gn0 + n, n == N - 1 ? qb : -1, dq);
            for (int n = 0; n < N; ++n) {
                const int gn = gn0 + n;
                const int b = gn % NSB, vs = gn % L::VST;
                if (lane == 0) KTRACE(10, gn);
                MMA_WAIT(bar(L::B_VF + vs), (gn / L::VST) & 1);
                if (lane == 0) KTRACE(11, gn);
                wait_softmax(L::B_PF + b, (gn / NSB) & 1);
                if (n == 0 && n_units_done > 0) wait_softmax(L::B_OE, (n_units_done - 1) & 1);  // O drained
                tc_fence_after();
                if (elect_one()) {
                    KTRACE(8, gn);
                    issue_pv(vs, b, n > 0);
                    commit(L::B_VE + vs);  // V stage free; O includes PV(gn)
                    if (n == N - 1) commit(L::B_OF);
                }
                __syncwarp();
                if (n + NSB < N) {
                    issue_s(gn + NSB, n + NSB == N - 1 ? qb : -1, dq);  // into the buffer P(gn) just left
                }
            }
            gn0 += N;
            ++n_units_done;
        }
    } else if (warp < 4 * NG) {
        // ========= softmax group g (tiles gn = g, g+2, ... over all units): thread = one query row =========
#if CDSP_REGSPLIT
        asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(CDSP_SOFTMAX_REGS) : "memory");
#endif
        const int g = warp >> 2;
        const int quad = warp & 3;  // TMEM lane quadrant
        const int r = quad * 32 + lane;
        const uint32_t lane_off = static_cast<uint32_t>(quad * 32) << 16;
        const uint32_t tO = tmem + lane_off + COL_O;
        float* msh = reinterpret_cast<float*>(smem + L::OFF_M);  // [2][BM]
        const float sl2 = p.scale_log2;
        volatile int* role_sh = reinterpret_cast<volatile int*>(smem + L::OFF_ROLE);  // [NG]
        int gn0 = 0, n_units_done = 0;
        for (int i = 0;; ++i) {
            const int ub = i & 1;
            mbar_wait(bar(L::B_UF + ub), (i >> 1) & 1);
            const UnitInfo u = uinfo[ub];
            if (u.x < 0) break;
            const int N = u.n_used;
            int head;
            int64_t row0;
            unit_rows(u.x, crank, head, row0);
            const int64_t row = row0 + r;
            const bool row_ok = row < nq;
            const uint16_t* list = reinterpret_cast<const uint16_t*>(smem + L::OFF_SCHED) + ub * L::LISTMAX;
            const int64_t* qp = reinterpret_cast<const int64_t*>(smem + L::OFF_QP) + ub * BM;

            float m = -INFINITY;       // m(n) of the last tile this thread has seen
            float m_used = -INFINITY;  // max that this group's l is relative to
            float2 lacc = make_float2(0.f, 0.f);
            // this group's tiles: tile gn of the CTA's sequence belongs to group gn mod NG
            const int n_first = ((g - gn0) % NG + NG) % NG;
            for (int n = n_first; n < N; n += NG) {
                const int gn = gn0 + n;
                const uint32_t e = list[n];
                const int j = static_cast<int>(e & ~kPartialBit);  // launch-global tile id
                const bool partial = (e & kPartialBit) != 0;
                const int b = gn % NSB;
                const uint32_t tS = tmem + lane_off + col_s(b);
                if (lane == 0 && quad == 0) KTRACE(12 + g, gn);
                mbar_wait(bar(L::B_SF + b), (gn / NSB) & 1);
                if (lane == 0 && quad == 0) KTRACE(4 * g + 0, gn);
                tc_fence_after();
#if defined(CDSP_DBG_SOFTMAX) && CDSP_DBG_SOFTMAX == 0
                // debug: MMA pipeline alone (no TMEM traffic from the softmax; results garbage)
                if (n > 0) named_bar_sync(2 + (gn - 1) % NG, 2 * BM);
                if (n < N - 1) named_bar_arrive(2 + gn % NG, 2 * BM);
                tc_fence_before();
                __syncwarp();
                if (lane == 0) arrive_leader(L::B_PF + b);
                continue;
#endif
                // 64 score registers: columns 64-127 first (max only), then 0-63 (max, kept for the
                // exponentials); 64-127 are re-read from TMEM for their exponentials (P(n) only ever
                // overwrites S columns 0-63)
#if CDSP_FULL_ROW
                // the whole score row in registers: one TMEM round trip, no re-reads
                uint32_t s[128];
                tmem_ld32p(tS, s);
                tmem_ld32p(tS + 32, s + 32);
                tmem_ld32p(tS + 64, s + 64);
                tmem_ld32p(tS + 96, s + 96);
                tc_wait_ld();
                reg_tie32(s);
                reg_tie32(s + 32);
                reg_tie32(s + 64);
                reg_tie32(s + 96);
                if (partial) mask_tile<4>(s, segs, toff, j, qp[r], 0);
                const float mx = fmaxf(max64(s), max64(s + 64)) * sl2;
#else
                uint32_t s[64];
                tmem_ld32p(tS + 64, s);
                tmem_ld32p(tS + 96, s + 32);
                tc_wait_ld();
                reg_tie32(s);
                reg_tie32(s + 32);
                if (partial) mask_tile<2>(s, segs, toff, j, qp[r], 64);
                const float mx_hi = max64(s);
                tmem_ld32p(tS, s);
                tmem_ld32p(tS + 32, s + 32);
                tc_wait_ld();
                reg_tie32(s);
                reg_tie32(s + 32);
                if (partial) mask_tile<2>(s, segs, toff, j, qp[r], 0);
                const float mx = fmaxf(mx_hi, max64(s)) * sl2;
#endif
#ifdef CDSP_KTRACE
                if (r == 0 && n == 0) UNIT_STAMP(u.x * CL + crank, 5, gtime_ns());
#endif
                // ---- the serial link: m(n) = lazy max(m(n-1), rowmax(S(n))) ----
                if (n > 0) {  // m(n-1) from the group of tile n-1 (named barrier 2 + its index: 128 + 128 threads)
                    named_bar_sync(2 + (gn - 1) % NG, 2 * BM);
                    m = msh[((gn - 1) % NG) * BM + r];
                }
                const bool need = mx > m + 8.0f;
                const float m_prev = m;
                if (need) m = mx;
                if (lane == 0 && quad == 0) KTRACE(4 * g + 1, gn);
                // O holds PV up to n-1 relative to m(n-1): rescale it once PV(n-1) completed, before
                // m(n) is published (so no later PV can be issued meanwhile)
                if (n > 0 && __any_sync(0xFFFFFFFFu, need)) {
                    mbar_wait(bar(L::B_VE + (gn - 1) % L::VST), ((gn - 1) / L::VST) & 1);  // PV(n-1) done
                    tc_fence_after();
                    const float alpha = need ? ex2(m_prev - m) : 1.0f;
#pragma unroll 1
                    for (int c = 0; c < HD / 16; ++c) {
                        uint32_t o[16];
                        tmem_ld16(tO + 16 * c, o);
                        tc_wait_ld();
                        reg_tie16(o);
#pragma unroll
                        for (int q = 0; q < 16; ++q) o[q] = __float_as_uint(__uint_as_float(o[q]) * alpha);
                        tmem_st16(tO + 16 * c, o);
                    }
                }
                if (n < N - 1) {  // (the unit's last m stays with its group, which finishes the unit)
                    msh[(gn % NG) * BM + r] = m;
                    __threadfence_block();
                    named_bar_arrive(2 + gn % NG, 2 * BM);
                }
                // the exponentials below must not be hoisted above the arrive (the other group
                // waits for m(n)): tie their inputs to a volatile asm after it
                reg_tie32(s);
                reg_tie32(s + 32);
#if CDSP_FULL_ROW
                reg_tie32(s + 64);
                reg_tie32(s + 96);
#endif
                asm volatile("" : "+f"(m));
#if defined(CDSP_DBG_SOFTMAX) && CDSP_DBG_SOFTMAX == 1
                // debug: S read + row max only, no exponentials / P stores
                tc_fence_before();
                __syncwarp();
                if (lane == 0) arrive_leader(L::B_PF + b);
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
#if CDSP_FULL_ROW
                exp32_store(s, sc, nm, lacc, tS);
                exp32_store(s + 32, sc, nm, lacc, tS + 16);
                exp32_store(s + 64, sc, nm, lacc, tS + 32);
                exp32_store(s + 96, sc, nm, lacc, tS + 48);
#else
                exp32_store(s, sc, nm, lacc, tS);
                tmem_ld32p(tS + 64, s);
                exp32_store(s + 32, sc, nm, lacc, tS + 16);
                tc_wait_ld();
                reg_tie32(s);
                tmem_ld32p(tS + 96, s + 32);
                if (partial) mask_tile<1>(s, segs, toff, j, qp[r], 64);
                exp32_store(s, sc, nm, lacc, tS + 32);
                tc_wait_ld();
                reg_tie32(s + 32);
                if (partial) mask_tile<1>(s + 32, segs, toff, j, qp[r], 96);
                exp32_store(s + 32, sc, nm, lacc, tS + 48);
#endif
                if (lane == 0 && quad == 0) KTRACE(4 * g + 2, gn);
                tc_wait_st();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) arrive_leader(L::B_PF + b);
                if (lane == 0 && quad == 0) KTRACE(4 * g + 3, gn);
            }
            __syncwarp();
            if (ARRIVE_LANE) mbar_arrive(bar(L::B_UE + ub));  // done with the unit's schedule / positions
#if CDSP_EPI_WARPS
            // hand this group's row statistics to the epilogue group: (the max the row sum is
            // relative to, the row sum); the group of the unit's last tile holds the final max
            if (N > 0) {
                const int pu = n_units_done & 1, use = n_units_done >> 1;
                float2* lsh = reinterpret_cast<float2*>(smem + L::OFF_L) + pu * NG * BM;
                if (use >= 1) mbar_wait(bar(L::B_LE + pu), (use - 1) & 1);  // slot read by the unit 2 back
                lsh[g * BM + r] = make_float2(m_used, lacc.x + lacc.y);
                __syncwarp();
                if (ARRIVE_LANE) mbar_arrive(bar(L::B_LF + pu));
                gn0 += N;
                ++n_units_done;
            }
        }
    } else if (CDSP_EPI_WARPS && warp < W_EPI0 + NEPI) {
        // ========= epilogue group: finishes every unit in order (one thread = one query row) =========
        asm volatile("setmaxnreg.dec.sync.aligned.u32 112;" ::: "memory");
        const int quad = warp & 3;  // TMEM lane quadrant
        const int r = quad * 32 + lane;
        const int g = 0;  // (named barriers / role slot of the epilogue group)
        const uint32_t lane_off = static_cast<uint32_t>(quad * 32) << 16;
        const uint32_t tO = tmem + lane_off + COL_O;
        volatile int* role_sh = reinterpret_cast<volatile int*>(smem + L::OFF_ROLE);
        const int stage_bar = 8 + NG;
        const unsigned stage_lead = static_cast<unsigned>(W_EPI0 * 32);
        int gn0 = 0, n_units_done = 0;
        for (int i = 0;; ++i) {
            const int ub = i & 1;
            mbar_wait(bar(L::B_UF + ub), (i >> 1) & 1);
            const UnitInfo u = uinfo[ub];
            __syncwarp();
            if (ARRIVE_LANE) mbar_arrive(bar(L::B_UE + ub));  // only the unit id and tile count are needed
            if (u.x < 0) break;
            const int N = u.n_used;
            int head, part, ux, b0_unused, b1_unused;
            int64_t row0;
            unit_map(u.x, crank, head, row0, part, ux, b0_unused, b1_unused);
            const int64_t row = row0 + r;
            const bool row_ok = row < nq;
            const int E = N > 0 ? (gn0 + N - 1) % NG : 0;
            float l = 0.f, m = -INFINITY;
            if (N > 0) {  // combine the groups' row sums relative to the final max (the last tile's group)
                const int pu = n_units_done & 1, use = n_units_done >> 1;
                const float2* lsh = reinterpret_cast<const float2*>(smem + L::OFF_L) + pu * NG * BM;
                mbar_wait(bar(L::B_LF + pu), use & 1);
                m = lsh[E * BM + r].x;
                if (m != -INFINITY) {  // (m = -inf: no visible key; the FMA-pipe exp2 floors at 2^-126)
#pragma unroll
                    for (int gg = 0; gg < NG; ++gg) {
                        const float2 ml = lsh[gg * BM + r];
                        if (ml.y > 0.f) l += gg == E ? ml.y : ml.y * ex2(ml.x - m);
                    }
                }
                __syncwarp();
                if (ARRIVE_LANE) mbar_arrive(bar(L::B_LE + pu));
                gn0 += N;
                ++n_units_done;
            }
            if (N == 0 && p.mode == CDSP_ATTN_MID && part < 0) continue;  // merging an empty block is the identity
            asm volatile("griddepcontrol.wait;" ::: "memory");
            bool split_first = false;
            int* scnt = nullptr;
            if (part >= 0) {
                scnt = p.split_cnt + 2 * (2 * ux + crank);
                split_first = split_role(scnt, role_sh, 12, BM, r == 0) != 0;
            }
            // the staging boxes: the previous unit's TMA store has read them
            if (threadIdx.x == stage_lead) bulk_wait_read0();
            named_bar_sync(stage_bar, BM);
            if (part < 0) run_epilogue(IntC<2>{}, IntC<2>{}, head, row0, row, row_ok, r, quad, N, l, m, n_units_done, tO, stage_bar, stage_lead, 0, HD / 64, true, true);
            else if (split_first) run_epilogue(IntC<0>{}, IntC<1>{}, head, row0, row, row_ok, r, quad, N, l, m, n_units_done, tO, stage_bar, stage_lead, 0, HD / 64, true, true);
            else run_epilogue(IntC<1>{}, IntC<0>{}, head, row0, row, row_ok, r, quad, N, l, m, n_units_done, tO, stage_bar, stage_lead, 0, HD / 64, true, true);
            if (split_first) {  // publish the partial (every thread's stores, then one release)
                __threadfence();
                named_bar_sync(12, BM);
                if (r == 0) asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(scnt + 1), "r"(1) : "memory");
            }
        }
    }
#else
#ifdef CDSP_KTRACE
            if (r == 0 && g == 0) UNIT_STAMP(u.x * CL + crank, 6, gtime_ns());
#endif
            // split-unit part, derived again here rather than kept live through the tile loop
            // (register pressure of the softmax)
            int part = -1, ux = 0;
            if (p.split) {
                int xx = u.x, h2, b0, b1;
                int64_t r2;
                asm volatile("" : "+r"(xx));
                unit_map(xx, crank, h2, r2, part, ux, b0, b1);
            }
            if (N == 0 && p.mode == CDSP_ATTN_MID && part < 0) continue;  // merging an empty block is the identity

            // ---------------- epilogue: normalise, then write / LSE-merge (R3) ----------------
            // One group finishes the unit: the group E that computed its last tile (it holds the
            // final m; group 0 for a unit without tiles).  The other groups hand over their row
            // sums and start the next unit at once, so its first tiles run under this epilogue.
            const int E = N > 0 ? (gn0 + N - 1) % NG : 0;
            float l = 0.f;
            if (N > 0) {
                const int pu = n_units_done & 1, use = n_units_done >> 1;
                float2* lsh = reinterpret_cast<float2*>(smem + L::OFF_L) + pu * NG * BM;
                gn0 += N;
                ++n_units_done;
                if (g != E) {
                    if (use >= 1) mbar_wait(bar(L::B_LE + pu), (use - 1) & 1);  // slot read by the unit 2 back
                    lsh[g * BM + r] = make_float2(m_used, lacc.x + lacc.y);
                    __syncwarp();
                    if (ARRIVE_LANE) mbar_arrive(bar(L::B_LF + pu));
                    continue;
                }
                mbar_wait(bar(L::B_LF + pu), use & 1);
                if (m != -INFINITY) {  // (m = -inf: no visible key; the FMA-pipe exp2 floors at 2^-126)
                    l = lacc.x + lacc.y;  // relative to m: this group made the last m (m_used == m)
#pragma unroll
                    for (int gg = 0; gg < NG; ++gg) {
                        if (gg == g) continue;
                        const float2 ml = lsh[gg * BM + r];
                        if (ml.y > 0.f) l += ml.y * ex2(ml.x - m);
                    }
                }
                __syncwarp();
                if (ARRIVE_LANE) mbar_arrive(bar(L::B_LE + pu));
            } else if (g != E) {
                continue;
            }
            // the accumulator / output belong to the previous launch until it completes (a no-op
            // unless this grid was launched as its programmatic dependent)
            asm volatile("griddepcontrol.wait;" ::: "memory");
            // split unit: the first sub-unit to get here leaves its partial in the accumulator rows,
            // the second merges it (R3) and writes the output
            // split unit: the first sub-unit to get here leaves its partial in the accumulator rows,
            // the second merges it (R3) and writes the output.  The epilogue is instantiated per
            // role (merge / to_acc compile-time there): a per-unit runtime choice costs the
            // softmax hundreds of bytes of register spills.
            bool split_first = false;
            int* scnt = nullptr;
            const int stage_bar = 8 + g;
            const unsigned stage_lead = static_cast<unsigned>(g * BM);
            if (part >= 0) {
                scnt = p.split_cnt + 2 * (2 * ux + crank);
                split_first = split_role(scnt, role_sh + g, 12 + g, BM, r == 0) != 0;
            }
            if (part < 0) run_epilogue(IntC<2>{}, IntC<2>{}, head, row0, row, row_ok, r, quad, N, l, m, n_units_done, tO, stage_bar, stage_lead, 0, HD / 64, true, true);
            else if (split_first) run_epilogue(IntC<0>{}, IntC<1>{}, head, row0, row, row_ok, r, quad, N, l, m, n_units_done, tO, stage_bar, stage_lead, 0, HD / 64, true, true);
            else run_epilogue(IntC<1>{}, IntC<0>{}, head, row0, row, row_ok, r, quad, N, l, m, n_units_done, tO, stage_bar, stage_lead, 0, HD / 64, true, true);
            if (split_first) {  // publish the partial (every thread's stores, then one release)
                __threadfence();
                named_bar_sync(12 + g, BM);
                if (r == 0) asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(scnt + 1), "r"(1) : "memory");
            }
#ifdef CDSP_KTRACE
            if (r == 0) {
                const unsigned long long t = gtime_ns();
                unsigned smid;
                asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
                const int ux = u.x * CL + crank;
                UNIT_STAMP(ux, 7, t);
                UNIT_STAMP(ux, 1, t);
                UNIT_STAMP(ux, 2, smid);
                UNIT_STAMP(ux, 3, N);
            }
#endif
        }
    }
#endif

    // ---- teardown
    if (PAIR && (CDSP_EPI_WARPS ? threadIdx.x == W_EPI0 * 32 : (warp < 4 * NG && (threadIdx.x % BM) == 0)))
        bulk_wait_all0();  // staged output stores done
    tc_fence_before();
    if constexpr (PAIR) cluster_sync_all();  // no remote arrive / DSMEM access into a CTA that exits
    else __syncthreads();
    if (warp == W_MMA) {
        tc_fence_after();
        if constexpr (PAIR) tmem_dealloc2(tmem, 512);
        else tmem_dealloc(tmem, 512);
    }
    if (threadIdx.x == 0) {  // the last CTA out re-arms the unit counter for a later launch
        __threadfence();
        if (atomicAdd(p.claim + 1, 1) == static_cast<int>(gridDim.x) - 1) {
            atomicExch(p.claim, 0);
            atomicExch(p.claim + 1, 0);
        }
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
cdsp_status make_map(CUtensorMap* m, const void* base, int64_t T, int H, int D, int box_rows = 128) {
    EncodeTiledFn enc = get_encode_fn();
    CDSP_REQUIRE(enc != nullptr, CDSP_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    CDSP_REQUIRE((reinterpret_cast<uintptr_t>(base) & 15u) == 0, CDSP_ERR_INVALID,
                 "TMA base pointer must be 16-byte aligned");
    cuuint64_t dims[3] = {static_cast<cuuint64_t>(D), static_cast<cuuint64_t>(H),
                          static_cast<cuuint64_t>(T > 0 ? T : 1)};
    cuuint64_t strides[2] = {static_cast<cuuint64_t>(D) * 2, static_cast<cuuint64_t>(H) * D * 2};
    cuuint32_t box[3] = {64, 1, static_cast<cuuint32_t>(box_rows)};
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    CDSP_REQUIRE(r == CUDA_SUCCESS, CDSP_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", static_cast<int>(r));
    return CDSP_OK;
}

// Per-device kernel state, allocated once (attention_device_init, called by cdsp_comm_create;
// a comm-less first cdsp_attention_fwd* call on a device allocates it then):
//  * unit counters of the persistent kernel: one [claim, done] pair per launch, taken
//    round-robin from a zeroed ring (each launch's last CTA re-zeroes its pair; a pair is reused
//    only after kClaimSlots later launches, far more than can run concurrently);
//  * split-unit counters: a launch with S split units takes 4 S ints ([unit][2 CTAs][arrivals,
//    ready]) from a zeroed ring of kSplitRing ints (bump allocation; every pair is re-zeroed by
//    its second finisher, and a range is reused only after the ring wrapped, i.e. after at
//    least kSplitRing / (4 kSplitUnits) = 32 later split launches).
constexpr int kClaimSlots = 4096;
constexpr int kSplitUnits = 32768;  // split units per launch (more: the launch runs unsplit)
constexpr int64_t kSplitRing = 32ll * 4 * kSplitUnits;
struct DevState {
    int* ring = nullptr;
    int* split = nullptr;
    unsigned counter = 0;
    int64_t split_next = 0;
};
DevState g_dev[64];

cdsp_status device_state(DevState** out) {
    int dev = 0;
    CDSP_CUDA(cudaGetDevice(&dev));
    CDSP_REQUIRE(dev >= 0 && dev < 64, CDSP_ERR_CUDA, "device ordinal %d", dev);
    DevState& d = g_dev[dev];
    if (!d.ring) {
        CDSP_CUDA(cudaMalloc(reinterpret_cast<void**>(&d.ring), kClaimSlots * 2 * sizeof(int)));
        CDSP_CUDA(cudaMemset(d.ring, 0, kClaimSlots * 2 * sizeof(int)));
        CDSP_CUDA(cudaMalloc(reinterpret_cast<void**>(&d.split), kSplitRing * sizeof(int)));
        CDSP_CUDA(cudaMemset(d.split, 0, kSplitRing * sizeof(int)));
        CDSP_CUDA(cudaDeviceSynchronize());
    }
    *out = &d;
    return CDSP_OK;
}
cdsp_status claim_slot(int** out) {
    DevState* d = nullptr;
    CDSP_CHECK_STATUS(device_state(&d));
    *out = d->ring + 2 * (__atomic_fetch_add(&d->counter, 1u, __ATOMIC_RELAXED) % kClaimSlots);
    return CDSP_OK;
}

int sm_count() {
    static int n[64] = {};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
    if (n[dev] == 0 && cudaDeviceGetAttribute(&n[dev], cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) n[dev] = 148;
    return n[dev];
}

// KV tiles (BN keys) a query row range [r0, r1) touches in block b (b < 0: all blocks): history
// tiles, then the tiles of the key rows of each segment whose positions reach the range's
// largest query position.  Host-side estimate for unit weights (exact for unmasked rows).
int64_t unit_tiles(const cdsp_segments* seg, int nblk, int64_t r0, int64_t r1, int only_b) {
    int64_t qlo, qhi;
    bool any;
    seg_qrange(seg[0], r0, r1, qlo, qhi, any);
    if (!any) return 0;
    int64_t t = 0;
    for (int b = 0; b < nblk; ++b) {
        if (only_b >= 0 && b != only_b) continue;
        const cdsp_segments& s = seg[b];
        const int64_t st = s.pos_stride > 0 ? s.pos_stride : 1;
        auto upto = [&](int64_t pos0, int64_t len) -> int64_t {  // rows of a segment with pos <= qhi
            if (len <= 0 || qhi < pos0) return 0;
            const int64_t n = (qhi - pos0) / st + 1;
            return n < len ? n : len;
        };
        const int64_t e0 = s.kv_hist + s.kv_len0;
        const int64_t a_end = s.kv_hist + upto(s.kv_pos0, s.kv_len0);  // rows [0, a_end) used
        const int64_t b_len = upto(s.kv_pos1, s.nkv - e0);              // rows [e0, e0 + b_len) used
        const int64_t ta = (a_end + BN - 1) / BN;
        int64_t tb = 0;
        if (b_len > 0) {
            const int64_t j0 = e0 / BN, j1 = (e0 + b_len - 1) / BN;
            const int64_t shared = j0 < ta ? (ta - j0 < j1 - j0 + 1 ? ta - j0 : j1 - j0 + 1) : 0;
            tb = j1 - j0 + 1 - shared;
        }
        t += ta + tb;
    }
    return t;
}

template <int HD, bool PAIR>
cdsp_status launch_tc(const AttnArgs& a, cudaStream_t st) {
    using Lt = Layout<HD, PAIR>;
    auto kern = attn_tc_kernel<HD, PAIR>;
    static int max_groups = 0;  // co-resident CTA groups (PAIR: clusters of 2 need 2 SMs of one GPC)
    if (max_groups == 0) {
        CDSP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Lt::SMEM));
        if (PAIR) {
            cudaLaunchConfig_t cfg = {};
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = 2;
            at[0].val.clusterDim.y = 1;
            at[0].val.clusterDim.z = 1;
            cfg.gridDim = dim3(2 * sm_count(), 1, 1);
            cfg.blockDim = dim3(kThreads, 1, 1);
            cfg.dynamicSmemBytes = Lt::SMEM;
            cfg.attrs = at;
            cfg.numAttrs = 1;
            int n = 0;
            CDSP_CUDA(cudaOccupancyMaxActiveClusters(&n, kern, &cfg));
            max_groups = n > 0 ? n : sm_count() / 2;
        } else {
            max_groups = sm_count();
        }
    }
    CDSP_REQUIRE(a.nblk >= 1 && a.nblk <= kMaxBlk, CDSP_ERR_INVALID, "%d KV blocks (1..%d)", a.nblk, kMaxBlk);
    const cdsp_segments& s0 = a.seg[0];
    TcParams p;
    std::memset(&p, 0, sizeof(p));
    p.nblk = a.nblk;
    int64_t tiles = 0;
    for (int b = 0; b < a.nblk; ++b) {
        p.seg[b] = a.seg[b];
        p.tile_off[b] = static_cast<int>(tiles);
        tiles += (a.seg[b].nkv + BN - 1) / BN;
        CDSP_REQUIRE(tiles <= Lt::LISTMAX, CDSP_ERR_CAPACITY, "KV blocks of %lld tiles exceed %d per launch",
                     static_cast<long long>(tiles), Lt::LISTMAX);
    }
    for (int b = a.nblk; b <= kMaxBlk; ++b) p.tile_off[b] = static_cast<int>(tiles);
    p.gate = a.gate;
    p.gate_target = a.gate_target;
    p.gate_mask = a.gate ? a.gate_mask : 0u;
    p.gate_ng = a.gate_ng > 0 ? a.gate_ng : 1;
    p.gate_hpg = a.gate_hpg > 0 ? a.gate_hpg : 1;
    p.gate_err = a.gate_err;
    p.Hq = a.Hq;
    p.Hkv = a.Hkv;
    p.g = a.Hq / a.Hkv;
    p.n_rb = static_cast<int>((s0.nq + BM - 1) / BM);
    p.n_pb = PAIR ? (p.n_rb + 1) / 2 : p.n_rb;
    static const int split_env = getenv("CDSP_SPLIT") ? atoi(getenv("CDSP_SPLIT")) : 1;
    static const int light_env = getenv("CDSP_LIGHT_LAST") ? atoi(getenv("CDSP_LIGHT_LAST")) : 1;
    DevState* dst = nullptr;
    CDSP_CHECK_STATUS(device_state(&dst));
    p.split = 0;
    p.split_blk = (a.nblk + 1) / 2;
    p.n_light = 0;
    p.heads_a = a.Hq;
    if (p.n_pb > 1 && (light_env || split_env)) {
        // unit weights (KV tiles) per row block; non-decreasing in pb (a row's keys grow with
        // its position)
        std::vector<int64_t> w(p.n_pb);
        int64_t W = 0;
        for (int pb = 0; pb < p.n_pb; ++pb) {
            w[pb] = unit_tiles(a.seg, a.nblk, static_cast<int64_t>(pb) * (PAIR ? 2 : 1) * BM,
                               static_cast<int64_t>(pb + 1) * (PAIR ? 2 : 1) * BM, -1);
            W += w[pb];
        }
        const int64_t wmax = w[p.n_pb - 1];
        // light units (they go last and fill the tail): under 1/4 of the heaviest on a ring launch
        // (its lower row blocks see few blocks: KTRACE s=8 rank 2 tail 134 -> 26 us), under 1/8
        // for one causal block (smaller tail pieces: s=1 tail 22 vs 45 us)
        const int light_div = a.nblk > 1 ? 4 : 8;
        if (light_env)
            while (p.n_light < p.n_pb - 1 && w[p.n_light] * light_div < wmax) ++p.n_light;
        int64_t w_light = 0, w_heavy = 0;  // per head
        for (int pb = 0; pb < p.n_pb; ++pb) (pb < p.n_light ? w_light : w_heavy) += w[pb];
        // split (ONLY-mode multi-block launches with scratch): units heavier than a sixth of a CTA
        // group's share, in the heads of the last ~1.5 waves, at the block boundary that halves
        // the heaviest unit
        const double share = static_cast<double>(W) * a.Hq / max_groups;
        // only where units are few per CTA group (the tail is a large part of the launch): 32K MHA
        // ring proxy, s = 8 (7 units per group) 1292-1294 split vs 1232-1237 TF/s; s = 4 (14) even;
        // s = 2 (28) no gain (profiles/r02_split_rule_ab.md)
        const bool few_units = static_cast<int64_t>(p.n_pb) * a.Hq < 10ll * max_groups;
        int n = 0;
        if (split_env && few_units && a.split_ok && a.nblk >= 2 && a.mode == CDSP_ATTN_ONLY && a.o_acc && a.lse_acc)
            while (n < p.n_pb - p.n_light && w[p.n_pb - 1 - n] * 6.0 > share && w[p.n_pb - 1 - n] >= 32) ++n;
        if (n > 0) {
            // region B + C (pieces no larger than half the heaviest unit) carries at least 1.5
            // heaviest units of work per CTA group: whatever region A's units leave uneven
            const double need = 1.5 * max_groups * static_cast<double>(wmax) - static_cast<double>(w_light) * a.Hq;
            int hb = need <= 0.0 ? 1 : static_cast<int>(need / static_cast<double>(w_heavy > 0 ? w_heavy : 1)) + 1;
            if (split_env >= 2) hb = a.Hq;  // CDSP_SPLIT=2: split in every head (measurement)
            if (hb > a.Hq) hb = a.Hq;
            if (static_cast<int64_t>(hb) * n <= kSplitUnits) {
                p.split = n;
                p.heads_a = a.Hq - hb;
                const int64_t top0 = static_cast<int64_t>(p.n_pb - 1) * (PAIR ? 2 : 1) * BM;
                const int64_t top1 = static_cast<int64_t>(p.n_pb) * (PAIR ? 2 : 1) * BM;
                int64_t acc = 0, best_d = INT64_MAX;
                int best = 1;
                for (int b = 0; b + 1 < a.nblk; ++b) {
                    acc += unit_tiles(a.seg, a.nblk, top0, top1, b);
                    const int64_t d = acc * 2 - wmax < 0 ? wmax - acc * 2 : acc * 2 - wmax;
                    if (d < best_d) {
                        best_d = d;
                        best = b + 1;
                    }
                }
                p.split_blk = best;
                const int64_t need = 4ll * hb * n;
                if (dst->split_next + need > kSplitRing) dst->split_next = 0;
                p.split_cnt = dst->split + dst->split_next;
                dst->split_next += need;
            }
        }
    }
    const int64_t units = static_cast<int64_t>(p.n_pb) * a.Hq + static_cast<int64_t>(p.split) * (a.Hq - p.heads_a);
    if (units == 0) return CDSP_OK;
    CDSP_REQUIRE(units < (1ll << 30), CDSP_ERR_SHAPE, "too many query tiles");
    p.n_units = static_cast<int>(units);
    p.scale_log2 = a.scale * 1.4426950408889634f;
    p.mode = a.mode;
    p.o_acc = a.o_acc;
    p.lse_acc = a.lse_acc;
    p.out = static_cast<__nv_bfloat16*>(a.out);
    p.lse = a.lse;
    CDSP_CHECK_STATUS(claim_slot(&p.claim));
    TcMaps tm;
    std::memset(&tm, 0, sizeof(tm));
    CDSP_CHECK_STATUS(make_map(&tm.q, a.q, s0.nq, a.Hq, HD));
    for (int b = 0; b < a.nblk; ++b) {
        const bool has = a.seg[b].nkv > 0;
        const void* kb = has ? a.k[b] : a.q;  // nkv == 0: map never dereferenced
        const void* vb = has ? a.v[b] : a.q;
        // PAIR: each CTA loads 64 of a K tile's 128 keys (and 64 of V's 128 d columns)
        CDSP_CHECK_STATUS(make_map(&tm.k[b], kb, a.seg[b].nkv, has ? a.Hkv : a.Hq, HD, PAIR ? BN / 2 : BN));
        CDSP_CHECK_STATUS(make_map(&tm.v[b], vb, a.seg[b].nkv, has ? a.Hkv : a.Hq, HD));
    }
    tm.out = tm.q;  // bf16 output (staged epilogue); never dereferenced in fp32-result modes
    if (PAIR && (a.mode == CDSP_ATTN_ONLY || a.mode == CDSP_ATTN_LAST))
        CDSP_CHECK_STATUS(make_map(&tm.out, a.out, s0.nq, a.Hq, HD));
    // persistent: one CTA per SM (TMEM and shared memory admit one), units claimed dynamically;
    // spare_sms leaves SMs to kernels this launch waits on (gated blocks copied by SM kernels)
    int cap_groups = max_groups - (a.spare_sms + (PAIR ? 1 : 0)) / (PAIR ? 2 : 1);
    if (cap_groups < 1) cap_groups = 1;
    const int groups = static_cast<int>(units < cap_groups ? units : cap_groups);
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = PAIR ? 2 : 1;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3(static_cast<unsigned>(groups * (PAIR ? 2 : 1)), 1, 1);
    cfg.blockDim = dim3(kThreads, 1, 1);
    cfg.dynamicSmemBytes = Lt::SMEM;
    cfg.stream = st;
    // MID / LAST steps of an internal ring chain depend on the previous launch only through the
    // accumulator, read and written after griddepcontrol.wait, so they may be launched as
    // programmatic dependents and start under its tail (CDSP_PDL=0: plain stream order,
    // measurement control)
    static const bool pdl_env = !(getenv("CDSP_PDL") != nullptr && getenv("CDSP_PDL")[0] == '0');
    int na = 0;
    if (PAIR) at[na++] = at[0];
    if (a.pdl && pdl_env && (a.mode == CDSP_ATTN_MID || a.mode == CDSP_ATTN_LAST)) {
        at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[na].val.programmaticStreamSerializationAllowed = 1;
        ++na;
    }
    cfg.attrs = at;
    cfg.numAttrs = na;
#ifdef CDSP_KTRACE
    if (getenv("CDSP_TRACE")) {  // debug builds: a clean per-unit record for this launch
        void* gc = nullptr;
        CDSP_CUDA(cudaGetSymbolAddress(&gc, g_cta));
        CDSP_CUDA(cudaMemsetAsync(gc, 0, sizeof(unsigned long long) * 65536 * 8, st));
    }
#endif
    CDSP_CUDA(cudaLaunchKernelEx(&cfg, kern, tm, p));
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

// [rows, H, D] bf16 tensor map (128-byte swizzle, box box_rows x 1 head x 64 d) for other kernels
cdsp_status make_tile_map(CUtensorMap* m, const void* base, int64_t rows, int H, int D, int box_rows) {
    return make_map(m, base, rows, H, D, box_rows);
}

cdsp_status attention_device_init() {
    DevState* d = nullptr;
    return device_state(&d);
}

int attention_tc_max_tiles(int D) {
    static const bool no_pair = getenv("CDSP_ATTN_1SM") != nullptr;
    int n = D == 128 ? (no_pair ? Layout<128, false>::LISTMAX : Layout<128, true>::LISTMAX) : Layout<64, false>::LISTMAX;
    // test knob: a smaller per-launch tile budget makes small rings take the multi-launch path
    if (const char* e = getenv("CDSP_MAX_TILES")) {
        const int m = atoi(e);
        if (m >= 1 && m < n) n = m;
    }
    return n;
}

cdsp_status launch_attention_tc(const AttnArgs& a, cudaStream_t st) {
#ifndef CDSP_NO_PAIR
    static const bool no_pair = getenv("CDSP_ATTN_1SM") != nullptr;  // measurement control: 1-SM kernel
#else
    const bool no_pair = true;
#endif
    if (a.D == 128) return no_pair ? launch_tc<128, false>(a, st) : launch_tc<128, true>(a, st);
    if (a.D == 64) return launch_tc<64, false>(a, st);
    CDSP_FAIL(CDSP_ERR_SHAPE, "head dim %d not supported (64 or 128)", a.D);
}

}  // namespace cdsp
