// plan.h — host-side CDSP plan logic (validation, zigzag geometry, cache balancing).
#pragma once

#include <cstdint>

#include "cdsp.h"

namespace cdsp {

// Everything one chunk's execution needs, derived from the plan alone (every rank of the
// group derives the same values, so no metadata crosses the network).
struct ChunkInfo {
    int c;           // chunk index
    int s, s_prev;   // SP size of this chunk / the previous one (s_prev = 0 for chunk 0)
    int64_t L, m;    // chunk length, zigzag shard length L / 2s
    int64_t C;       // global position of the chunk's first token (= earlier tokens)
    int interleave;  // cdsp_interleave of this chunk
    int32_t ranks[CDSP_MAX_SP];         // ring order (instance ids)
    int64_t store_before[CDSP_MAX_SP];  // store rows held after chunk c-1 (0 for new ranks)
    int64_t hist[CDSP_MAX_SP];          // store rows after balancing = history seen by this chunk
    int n_moves;
    cdsp_move moves[CDSP_MAX_SP];
};

// Validate the whole plan (R9) and fill `info` for chunk c.
cdsp_status plan_chunk_info(const cdsp_plan* plan, int c, ChunkInfo* info);

// Ring rank of instance `inst` in the chunk, or -1.
int plan_ring_rank(const ChunkInfo& ci, int inst);

// Global positions of ring rank r's shard rows, st = shard_stride: rows [0, m) -> pos0 + i st,
// rows [m, 2m) -> pos1 + (i - m) st.  Zigzag: S_r then S_{2s-1-r} (st = 1); striped: tokens
// r, r + s, ... (st = s, pos1 = pos0 + m s continues the same stripe sequence).
inline int64_t shard_stride(const ChunkInfo& ci) { return ci.interleave == CDSP_STRIPED ? ci.s : 1; }
inline int64_t shard_pos0(const ChunkInfo& ci, int r) {
    return ci.interleave == CDSP_STRIPED ? ci.C + r : ci.C + static_cast<int64_t>(r) * ci.m;
}
inline int64_t shard_pos1(const ChunkInfo& ci, int r) {
    return ci.interleave == CDSP_STRIPED ? ci.C + r + ci.m * ci.s
                                         : ci.C + static_cast<int64_t>(2 * ci.s - 1 - r) * ci.m;
}

// Largest (history + shard) any rank holds over the plan: the store capacity it needs.
int64_t plan_max_store(const cdsp_plan* plan);

}  // namespace cdsp
