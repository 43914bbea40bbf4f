// attn_common.cuh — position/segment masking and the LSE-merge epilogue arithmetic shared
// by the two block-attention kernels (tcgen05 bf16, FFMA fp32).
//
// Mask ("each token ... all previous tokens", "each chunk computes attention
// with all historical tokens", readings R4/R5): KV row c is visible to a query at global
// position t iff c is history (c < kv_hist) or pos(c) <= t.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "cdsp.h"

namespace cdsp {

enum TileKind : int { TILE_EMPTY = 0, TILE_FULL = 1, TILE_PARTIAL = 2 };

// Positions step by pos_stride (1 zigzag / contiguous, s striped; cdsp.h).
__host__ __device__ __forceinline__ int64_t seg_qpos(const cdsp_segments& s, int64_t i) {
    return i < s.q_len0 ? s.q_pos0 + i * s.pos_stride : s.q_pos1 + (i - s.q_len0) * s.pos_stride;
}

// Min / max global position of valid query rows [r0, r1) (clipped to nq).  any=false: no rows.
__host__ __device__ __forceinline__ void seg_qrange(const cdsp_segments& s, int64_t r0, int64_t r1,
                                                    int64_t& lo, int64_t& hi, bool& any) {
    if (r1 > s.nq) r1 = s.nq;
    lo = INT64_MAX;
    hi = INT64_MIN;
    any = false;
    const int64_t a0 = r0, a1 = r1 < s.q_len0 ? r1 : s.q_len0;  // segment 0 part
    const int64_t st = s.pos_stride;
    if (a0 < a1) {
        any = true;
        lo = s.q_pos0 + a0 * st;
        hi = s.q_pos0 + (a1 - 1) * st;
    }
    const int64_t b0 = r0 > s.q_len0 ? r0 : s.q_len0, b1 = r1;  // segment 1 part
    if (b0 < b1) {
        any = true;
        const int64_t l1 = s.q_pos1 + (b0 - s.q_len0) * st, h1 = s.q_pos1 + (b1 - 1 - s.q_len0) * st;
        lo = l1 < lo ? l1 : lo;
        hi = h1 > hi ? h1 : hi;
    }
}

// Classify KV tile [c0, c0 + bn) against a query tile with position range [qlo, qhi].
__host__ __device__ __forceinline__ int seg_tile_kind(const cdsp_segments& s, bool qany, int64_t qlo,
                                                      int64_t qhi, int64_t c0, int bn) {
    if (!qany || c0 >= s.nkv) return TILE_EMPTY;
    const int64_t c1 = (c0 + bn < s.nkv) ? c0 + bn : s.nkv;
    const bool has_hist = c0 < s.kv_hist;
    int64_t kmin = INT64_MAX, kmax = INT64_MIN;
    const int64_t e0 = s.kv_hist + s.kv_len0;
    {  // segment 0 rows [max(c0,hist), min(c1,e0))
        const int64_t a = c0 > s.kv_hist ? c0 : s.kv_hist, b = c1 < e0 ? c1 : e0;
        if (a < b) {
            kmin = s.kv_pos0 + (a - s.kv_hist) * s.pos_stride;
            kmax = s.kv_pos0 + (b - 1 - s.kv_hist) * s.pos_stride;
        }
    }
    {  // segment 1 rows [max(c0,e0), c1)
        const int64_t a = c0 > e0 ? c0 : e0, b = c1;
        if (a < b) {
            const int64_t x0 = s.kv_pos1 + (a - e0) * s.pos_stride, x1 = s.kv_pos1 + (b - 1 - e0) * s.pos_stride;
            kmin = x0 < kmin ? x0 : kmin;
            kmax = x1 > kmax ? x1 : kmax;
        }
    }
    const bool has_seg = kmin <= kmax;
    if (!has_hist && has_seg && kmin > qhi) return TILE_EMPTY;
    const bool all_visible = (!has_seg || kmax <= qlo) && (c0 + bn <= s.nkv);
    return all_visible ? TILE_FULL : TILE_PARTIAL;
}

// Per-element visibility of KV row c for a query at position qpos.
__device__ __forceinline__ bool seg_visible(const cdsp_segments& s, int64_t c, int64_t qpos) {
    if (c >= s.nkv) return false;
    if (c < s.kv_hist) return true;
    const int64_t j = c - s.kv_hist;
    const int64_t kp = j < s.kv_len0 ? s.kv_pos0 + j * s.pos_stride : s.kv_pos1 + (j - s.kv_len0) * s.pos_stride;
    return kp <= qpos;
}

// LSE-merge weights (R3) for combining the running accumulator (lse_a) with a new block
// (lse_b), both natural-log; wa + wb normalises.  Both -inf: wa = wb = 0, lse = -inf.
__device__ __forceinline__ void merge_weights(float lse_a, float lse_b, float& wa, float& wb, float& lse) {
    const float M = fmaxf(lse_a, lse_b);
    if (M == -INFINITY) {
        wa = 0.f;
        wb = 0.f;
        lse = -INFINITY;
        return;
    }
    const float ea = __expf(lse_a - M), eb = __expf(lse_b - M);
    const float den = ea + eb;
    wa = ea / den;
    wb = eb / den;
    lse = M + __logf(den);
}

}  // namespace cdsp
