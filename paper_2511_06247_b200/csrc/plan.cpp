// plan.cpp — host-side CDSP plan logic.
//
// Plan format: A = [(token count, instance group)] (Alg. 1, D1).  Group rules
// (§4.1): "each chunk's instance group must include all instances involved in
// preceding chunks"; SP sizes are powers of two — reading R9: s in {1,2,4,8},
// non-decreasing, integral ratio, previous ring order is a prefix, ranks distinct; and
// R6: len % 2s == 0 (zigzag's 2N equal shards).
//
// Cache balancing ("the KV cache of all preceding chunks is evenly re-distributed
// to current chunk's instance group"; Fig. 5: "P0-P3 forward the second half of their
// local KV cache to P4-P7") — reading R8: with k = s_c / s_{c-1}, old ring rank i keeps the
// first of k contiguous store parts (sizes floor(n/k) + [j < n mod k]) and sends part j
// to ring rank i + j s_{c-1}.  Store sizes evolve as: balance, then += 2m (own shard).
#include "plan.h"

#include <cstring>

#include "common.cuh"

namespace cdsp {

namespace {
bool pow2_sp(int s) { return s == 1 || s == 2 || s == 4 || s == 8; }
}  // namespace

cdsp_status plan_chunk_info(const cdsp_plan* plan, int c, ChunkInfo* info) {
    CDSP_REQUIRE(plan && plan->chunks && info, CDSP_ERR_INVALID, "NULL plan/info");
    CDSP_REQUIRE(plan->n_chunks >= 1, CDSP_ERR_PLAN, "plan has no chunks");
    CDSP_REQUIRE(c >= 0 && c < plan->n_chunks, CDSP_ERR_INVALID, "chunk %d out of range [0,%d)", c,
                 plan->n_chunks);
    // validation of every chunk (a plan is legal or not as a whole)
    int max_inst = -1;
    for (int i = 0; i < plan->n_chunks; ++i) {
        const cdsp_chunk& ch = plan->chunks[i];
        CDSP_REQUIRE(ch.ranks != nullptr, CDSP_ERR_INVALID, "chunk %d: NULL ranks", i);
        CDSP_REQUIRE(ch.interleave == CDSP_ZIGZAG || ch.interleave == CDSP_STRIPED, CDSP_ERR_PLAN,
                     "chunk %d: interleave %d not zigzag (0) / striped (1)", i, ch.interleave);
        CDSP_REQUIRE(pow2_sp(ch.sp), CDSP_ERR_PLAN, "chunk %d: sp=%d not in {1,2,4,8}", i, ch.sp);
        CDSP_REQUIRE(ch.len > 0 && ch.len % (2 * static_cast<int64_t>(ch.sp)) == 0, CDSP_ERR_PLAN,
                     "chunk %d: len=%lld not a positive multiple of 2*sp", i, static_cast<long long>(ch.len));
        for (int a = 0; a < ch.sp; ++a) {
            CDSP_REQUIRE(ch.ranks[a] >= 0, CDSP_ERR_PLAN, "chunk %d: negative rank", i);
            if (ch.ranks[a] > max_inst) max_inst = ch.ranks[a];
            for (int b = 0; b < a; ++b)
                CDSP_REQUIRE(ch.ranks[a] != ch.ranks[b], CDSP_ERR_PLAN, "chunk %d: duplicate rank %d", i,
                             ch.ranks[a]);
        }
        if (i > 0) {
            const cdsp_chunk& pv = plan->chunks[i - 1];
            CDSP_REQUIRE(ch.sp >= pv.sp && ch.sp % pv.sp == 0, CDSP_ERR_PLAN,
                         "chunk %d: sp %d -> %d must grow by an integral factor", i, pv.sp, ch.sp);
            for (int a = 0; a < pv.sp; ++a)
                CDSP_REQUIRE(ch.ranks[a] == pv.ranks[a], CDSP_ERR_PLAN,
                             "chunk %d: group must extend chunk %d's ring order (P:155)", i, i - 1);
        }
    }
    // store sizes by ring position: ranks of chunk c' are a prefix of chunk c's, so ring
    // position k denotes the same instance throughout.
    int64_t size[CDSP_MAX_SP] = {0};
    int64_t C = 0;
    std::memset(info, 0, sizeof(*info));
    for (int i = 0; i <= c; ++i) {
        const cdsp_chunk& ch = plan->chunks[i];
        const int s = ch.sp, sp = i > 0 ? plan->chunks[i - 1].sp : 0;
        if (i == c) {
            info->c = c;
            info->s = s;
            info->s_prev = sp;
            info->L = ch.len;
            info->m = ch.len / (2 * s);
            info->C = C;
            info->interleave = ch.interleave;
            for (int r = 0; r < s; ++r) {
                info->ranks[r] = ch.ranks[r];
                info->store_before[r] = size[r];
            }
        }
        if (i > 0 && s > sp) {
            const int k = s / sp;
            int nm = 0;
            for (int r = 0; r < sp; ++r) {
                const int64_t n = size[r];
                int64_t off = 0;
                for (int j = 0; j < k; ++j) {
                    const int64_t part = n / k + (j < n % k ? 1 : 0);
                    if (j == 0) {
                        size[r] = part;
                    } else {
                        size[r + j * sp] = part;
                        if (i == c) info->moves[nm++] = cdsp_move{r, r + j * sp, off, part};
                    }
                    off += part;
                }
            }
            if (i == c) info->n_moves = nm;
        }
        if (i == c) {
            for (int r = 0; r < s; ++r) info->hist[r] = size[r];
            break;
        }
        for (int r = 0; r < s; ++r) size[r] += ch.len / s;  // own zigzag shard, 2m rows
        C += ch.len;
    }
    return CDSP_OK;
}

int plan_ring_rank(const ChunkInfo& ci, int inst) {
    for (int r = 0; r < ci.s; ++r)
        if (ci.ranks[r] == inst) return r;
    return -1;
}

int64_t plan_max_store(const cdsp_plan* plan) {
    int64_t best = 0;
    for (int c = 0; c < plan->n_chunks; ++c) {
        ChunkInfo ci;
        if (plan_chunk_info(plan, c, &ci) != CDSP_OK) return -1;
        for (int r = 0; r < ci.s; ++r) {
            const int64_t need = ci.hist[r] + 2 * ci.m;
            if (need > best) best = need;
        }
    }
    return best;
}

}  // namespace cdsp
