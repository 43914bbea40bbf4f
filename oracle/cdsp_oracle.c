/*
 * cdsp_oracle.c — the CPU ORACLE for the CDSP chunked-prefill ring-attention hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  The product path
 * (paper_2511_06247_b200/, libcdsp.so) never links, loads or calls it, and this file
 * shares no code, header, table or constant with the CUDA path.
 *
 * Plain, slow, obviously-correct C in float64.  Every function cites the passage of
 * /root/reference/PAPER.md ("P:<line>", section) it writes out, and the DESIGN.md
 * reading ("R<n>", = SURVEY.md §8(c) item n) it takes where the paper is silent.
 *
 *   oracle_attention        exact masked softmax attention (definition)
 *   oracle_causal_rows      the same over the whole unsharded prompt, for selected rows
 *   oracle_zigzag_map       zigzag 2N-shard partition, chunk-local (R5)
 *   oracle_striped_map      striped (round-robin) partition
 *   oracle_plan_stores      CDSP cache balancing + store contents per chunk (R8, R9)
 *   oracle_paged_write      decode paged-KV writer (R15)
 *   oracle_lse_merge        n-way log-sum-exp merge of partial attention (R3)
 *
 * Parity pins (what fixes each function independently of itself) live in
 * tests/test_oracle.py; see DESIGN.md §"Oracle and pins".
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORACLE_OK 0
#define ORACLE_ERR_ARG 1
#define ORACLE_ERR_PLAN 4
#define ORACLE_ERR_RANGE 5

int oracle_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/*
 * Exact attention of selected query rows over a key set, visible iff kpos[j] <= qpos[r].
 *
 * P:45 (§2.1): "self-attention requires each token to interact with all previous tokens'
 * key/value vectors"; P:59 (§2.3): each instance interacts "local query tensors with full
 * key-value tensors"; P:161 (§4.1): "each chunk computes attention with all historical
 * tokens".  The result is therefore plain softmax attention under the causal mask on
 * global positions (R4: key j = t is visible; R5: positions are global).
 *
 * Definition written out, for query row r (position t = qpos[r]) and Q head h,
 * kv = floor(h / g), g = Hq / Hkv (R14), sigma = scale (R1: caller passes 1/sqrt(D)):
 *     s_j   = sigma * <q_r,h , k_j,kv>                 for j with kpos[j] <= t
 *     lse   = ln sum_j exp(s_j)                         (R2: natural log)
 *     o_r,h = sum_j exp(s_j - lse) * v_j,kv
 * Rows with no visible key: lse = -inf, o = 0 (R16).
 *
 * Layouts: q [nq, Hq, D]; k, v [nk, Hkv, D] (D fastest), float32 storage (every bf16 and
 * fp32 input value is exact in float32), arithmetic in double.
 * Outputs: out [nq, Hq, D] double; lse [Hq, nq] double.
 */
int oracle_attention(const float* q, const int64_t* qpos, int64_t nq,
                     const float* k, const float* v, const int64_t* kpos, int64_t nk,
                     int Hq, int Hkv, int D, double scale, double* out, double* lse) {
    if (!q || !qpos || !out || !lse || nq < 0 || nk < 0 || Hq <= 0 || Hkv <= 0 || D <= 0)
        return ORACLE_ERR_ARG;
    if (nk > 0 && (!k || !v || !kpos)) return ORACLE_ERR_ARG;
    if (Hq % Hkv != 0) return ORACLE_ERR_ARG;
    const int g = Hq / Hkv;
    int rc = ORACLE_OK;
#pragma omp parallel
    {
        double* s = (double*)malloc(sizeof(double) * (size_t)(nk > 0 ? nk : 1));
        if (!s) {
#pragma omp atomic write
            rc = ORACLE_ERR_ARG;
        }
#pragma omp for collapse(2) schedule(dynamic, 4)
        for (int64_t r = 0; r < nq; ++r) {
            for (int h = 0; h < Hq; ++h) {
                if (!s) continue;
                const int kvh = h / g;
                const float* qr = q + ((size_t)r * Hq + h) * D;
                double* o = out + ((size_t)r * Hq + h) * D;
                const int64_t t = qpos[r];
                /* scores of the visible keys, and their maximum (for a stable ln-sum-exp) */
                double M = -INFINITY;
                for (int64_t j = 0; j < nk; ++j) {
                    if (kpos[j] > t) { s[j] = -INFINITY; continue; }
                    const float* kj = k + ((size_t)j * Hkv + kvh) * D;
                    double dot = 0.0;
                    for (int d = 0; d < D; ++d) dot += (double)qr[d] * (double)kj[d];
                    s[j] = scale * dot;
                    if (s[j] > M) M = s[j];
                }
                for (int d = 0; d < D; ++d) o[d] = 0.0;
                if (M == -INFINITY) {           /* nothing visible (R16) */
                    lse[(size_t)h * nq + r] = -INFINITY;
                    continue;
                }
                double sum = 0.0;
                for (int64_t j = 0; j < nk; ++j)
                    if (s[j] != -INFINITY) sum += exp(s[j] - M);
                const double l = M + log(sum);  /* = ln sum_j exp(s_j) */
                lse[(size_t)h * nq + r] = l;
                for (int64_t j = 0; j < nk; ++j) {
                    if (s[j] == -INFINITY) continue;
                    const double p = exp(s[j] - l);
                    const float* vj = v + ((size_t)j * Hkv + kvh) * D;
                    for (int d = 0; d < D; ++d) o[d] += p * (double)vj[d];
                }
            }
        }
        free(s);
    }
    return rc;
}

/*
 * The method's end result (north_star): causal attention over the WHOLE
 * unsharded prompt, independent of plan, SP sizes and chunking.
 * q, k, v are the full [N, H, D] tensors; rows[] selects which query positions to
 * evaluate (rows == NULL: all N).  out [n_rows, Hq, D], lse [Hq, n_rows].
 */
int oracle_causal_rows(const float* q, const float* k, const float* v, int64_t N,
                       int Hq, int Hkv, int D, double scale,
                       const int64_t* rows, int64_t n_rows, double* out, double* lse) {
    if (!q || !k || !v || N < 0) return ORACLE_ERR_ARG;
    if (!rows) n_rows = N;
    int64_t* qpos = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n_rows > 0 ? n_rows : 1));
    int64_t* kpos = (int64_t*)malloc(sizeof(int64_t) * (size_t)(N > 0 ? N : 1));
    float* qs = (float*)malloc(sizeof(float) * (size_t)(n_rows > 0 ? n_rows : 1) * Hq * D);
    if (!qpos || !kpos || !qs) { free(qpos); free(kpos); free(qs); return ORACLE_ERR_ARG; }
    int rc = ORACLE_OK;
    for (int64_t j = 0; j < N; ++j) kpos[j] = j;
    for (int64_t r = 0; r < n_rows; ++r) {
        const int64_t t = rows ? rows[r] : r;
        if (t < 0 || t >= N) { rc = ORACLE_ERR_RANGE; break; }
        qpos[r] = t;
        memcpy(qs + (size_t)r * Hq * D, q + (size_t)t * Hq * D, sizeof(float) * (size_t)Hq * D);
    }
    if (rc == ORACLE_OK)
        rc = oracle_attention(qs, qpos, n_rows, k, v, kpos, N, Hq, Hkv, D, scale, out, lse);
    free(qpos); free(kpos); free(qs);
    return rc;
}

/*
 * Zigzag partition, P:75 (§2.3): "partitions the sequence into 2N shards S_0..S_{2N-1}
 * for N SP instances, and allocates (S_i, S_{2N-i-1}) to instance i".  Applied to the
 * chunk-local token indices of one chunk ("each chunk's tokens are evenly
 * interleaved"; R5), N = s, shard length m = L / (2s) (R6: L % 2s == 0 required).
 *
 * tok_rank[t] = ring rank owning chunk-local token t; tok_slot[t] = its row in that
 * rank's shard, where the rank's shard lists S_i first, then S_{2s-1-i}.
 */
int oracle_zigzag_map(int64_t L, int s, int32_t* tok_rank, int32_t* tok_slot) {
    if (s <= 0 || L < 0 || (L % (2 * (int64_t)s)) != 0) return ORACLE_ERR_ARG;
    const int64_t m = L / (2 * (int64_t)s);
    for (int64_t t = 0; t < L; ++t) {
        const int64_t j = m > 0 ? t / m : 0;       /* shard index S_j */
        int32_t owner;
        int64_t slot;
        if (j < s) { owner = (int32_t)j; slot = t - j * m; }                 /* S_i        */
        else       { owner = (int32_t)(2 * s - 1 - j); slot = m + (t - j * m); } /* S_{2s-1-i} */
        if (tok_rank) tok_rank[t] = owner;
        if (tok_slot) tok_slot[t] = (int32_t)slot;
    }
    return ORACLE_OK;
}

/*
 * Striped partition, chunk-local.  P:75 (§2.3): "Striped Attention [5] partitions the
 * sequence into evenly-spaced stripes and assigns them to each instance in a round-robin
 * manner, so that each instance can conduct computation to every KV cache shard"; P:161:
 * "we can still adopt striped/zigzag attention to achieve intra-chunk attention load
 * balance".  Stripes of one token: token t belongs to instance t mod s and is row t / s
 * of its shard (reading R20; the chunk length rule R6, L % 2s == 0, is kept for both).
 */
int oracle_striped_map(int64_t L, int s, int32_t* tok_rank, int32_t* tok_slot) {
    if (s <= 0 || L < 0 || (L % (2 * (int64_t)s)) != 0) return ORACLE_ERR_ARG;
    for (int64_t t = 0; t < L; ++t) {
        if (tok_rank) tok_rank[t] = (int32_t)(t % s);   /* round-robin owner */
        if (tok_slot) tok_slot[t] = (int32_t)(t / s);   /* stripe index      */
    }
    return ORACLE_OK;
}

/*
 * CDSP store simulation: the plan A = [(token count, instance group)] (D1) is run
 * through P:155 (§4.1, Fig. 5): "each chunk's tokens are evenly interleaved across the
 * assigned prefill instance group.  All instance groups compute sequentially following
 * the chunk order.  Before computing each chunk, the KV cache of all preceding chunks is
 * evenly re-distributed to current chunk's instance group ... each chunk's instance
 * group must include all instances involved in preceding chunks".  Worked example:
 * "P0-P3 forward the second half of their local KV cache to P4-P7".
 *
 * Readings: R9 — s_c in {1,2,4,8} non-decreasing, s_c / s_{c-1} an integer
 * (a power of two), the previous group's ring order is a prefix of the next one's, ranks
 * distinct.  R8 — with k = s_c / s_{c-1}, old ring rank i splits its store (in store
 * order) into k contiguous parts, part j holding floor(n/k) + [j < n mod k] tokens; part 0
 * stays, part j moves to ring rank i + j*s_{c-1}.  Store order: chunk order, and within a
 * chunk the owner's zigzag shard order (S_i then S_{2s-1-i}); each chunk's shard is
 * appended after the history.
 *
 * Plan arrays: len[c], sp[c], ranks = concatenation of each chunk's ring order
 * (chunk c's list starts at sum_{c'<c} sp[c']).
 *
 * Output for chunk `upto` (the state right BEFORE chunk `upto` computes, after its
 * balancing):  store_n[i] = history tokens held by ring rank i of chunk `upto`;
 * store_pos[i * pos_stride + x] = their global positions in store order (may be NULL);
 * moves (may be NULL): up to 8 entries (src ring rank, dst ring rank, src offset, n_tok)
 * of chunk `upto`'s balancing; *n_moves their count.  Returns ORACLE_ERR_PLAN for an
 * illegal plan.
 */
int oracle_plan_stores_il(int n_chunks, const int64_t* len, const int32_t* sp, const int32_t* ranks,
                          const int32_t* interleave, int upto, int64_t* store_n, int64_t* store_pos,
                          int64_t pos_stride, int64_t* moves, int32_t* n_moves);

int oracle_plan_stores(int n_chunks, const int64_t* len, const int32_t* sp, const int32_t* ranks,
                       int upto, int64_t* store_n, int64_t* store_pos, int64_t pos_stride,
                       int64_t* moves, int32_t* n_moves) {
    return oracle_plan_stores_il(n_chunks, len, sp, ranks, NULL, upto, store_n, store_pos, pos_stride, moves,
                                 n_moves);
}

/* As oracle_plan_stores; interleave[c] (NULL: all zigzag) = 0 zigzag, 1 striped picks how
 * chunk c's tokens are interleaved ("striped/zigzag"), i.e. the shard appended. */
int oracle_plan_stores_il(int n_chunks, const int64_t* len, const int32_t* sp, const int32_t* ranks,
                          const int32_t* interleave, int upto, int64_t* store_n, int64_t* store_pos,
                          int64_t pos_stride, int64_t* moves, int32_t* n_moves) {
    if (n_chunks <= 0 || !len || !sp || !ranks || upto < 0 || upto >= n_chunks || !store_n)
        return ORACLE_ERR_ARG;
    /* validate the plan (R9) */
    int off = 0;
    int max_inst = -1;
    for (int c = 0; c < n_chunks; ++c) {
        const int s = sp[c];
        if (!(s == 1 || s == 2 || s == 4 || s == 8)) return ORACLE_ERR_PLAN;
        if (len[c] <= 0 || len[c] % (2 * (int64_t)s) != 0) return ORACLE_ERR_PLAN;
        for (int i = 0; i < s; ++i) {
            if (ranks[off + i] < 0) return ORACLE_ERR_PLAN;
            if (ranks[off + i] > max_inst) max_inst = ranks[off + i];
            for (int i2 = 0; i2 < i; ++i2)
                if (ranks[off + i2] == ranks[off + i]) return ORACLE_ERR_PLAN;
        }
        if (c > 0) {
            const int sprev = sp[c - 1];
            if (s < sprev || s % sprev != 0) return ORACLE_ERR_PLAN;
            const int offprev = off - sprev;
            for (int i = 0; i < sprev; ++i)
                if (ranks[offprev + i] != ranks[off + i]) return ORACLE_ERR_PLAN;
        }
        off += s;
    }
    /* stores, indexed by instance id; positions in store order */
    int64_t total = 0;
    for (int c = 0; c < n_chunks; ++c) total += len[c];
    const int n_inst = max_inst + 1;
    int64_t** st = (int64_t**)calloc((size_t)n_inst, sizeof(int64_t*));
    int64_t* stn = (int64_t*)calloc((size_t)n_inst, sizeof(int64_t));
    int64_t* tmp = (int64_t*)malloc(sizeof(int64_t) * (size_t)(total > 0 ? total : 1));
    if (!st || !stn || !tmp) { free(st); free(stn); free(tmp); return ORACLE_ERR_ARG; }
    for (int i = 0; i < n_inst; ++i) {
        st[i] = (int64_t*)malloc(sizeof(int64_t) * (size_t)(total > 0 ? total : 1));
        if (!st[i]) { for (int x = 0; x < i; ++x) free(st[x]); free(st); free(stn); free(tmp); return ORACLE_ERR_ARG; }
    }
    int rc = ORACLE_OK;
    int64_t C = 0;   /* historical tokens before chunk c */
    off = 0;
    int nm = 0;
    for (int c = 0; c <= upto; ++c) {
        const int s = sp[c];
        const int32_t* grp = ranks + off;
        /* 1. cache balancing onto this chunk's group (R8) */
        nm = 0;
        if (c > 0 && s > sp[c - 1]) {
            const int sprev = sp[c - 1];
            const int kk = s / sprev;
            for (int i = 0; i < sprev; ++i) {
                const int src = grp[i];
                const int64_t n = stn[src];
                memcpy(tmp, st[src], sizeof(int64_t) * (size_t)n);
                int64_t start = 0;
                for (int j = 0; j < kk; ++j) {
                    const int64_t part = n / kk + (j < n % kk ? 1 : 0);
                    if (j == 0) {
                        stn[src] = part;                 /* part 0 stays */
                    } else {
                        const int dst = grp[i + j * sprev];
                        memcpy(st[dst], tmp + start, sizeof(int64_t) * (size_t)part);
                        stn[dst] = part;
                        if (c == upto && moves && nm < 8) {
                            moves[nm * 4 + 0] = i;
                            moves[nm * 4 + 1] = i + j * sprev;
                            moves[nm * 4 + 2] = start;
                            moves[nm * 4 + 3] = part;
                        }
                        if (c == upto) ++nm;
                    }
                    start += part;
                }
            }
        }
        if (c == upto) break;
        /* 2. compute chunk c, then append each rank's zigzag shard to its store */
        const int64_t L = len[c];
        const int64_t m = L / (2 * (int64_t)s);
        const int striped = interleave && interleave[c] == 1;
        if (interleave && interleave[c] != 0 && interleave[c] != 1) { rc = ORACLE_ERR_PLAN; break; }
        for (int i = 0; i < s; ++i) {
            const int inst = grp[i];
            int64_t n = stn[inst];
            if (striped) {
                for (int64_t x = 0; x < L / s; ++x) st[inst][n++] = C + x * s + i;                 /* stripe x */
            } else {
                for (int64_t x = 0; x < m; ++x) st[inst][n++] = C + (int64_t)i * m + x;            /* S_i */
                for (int64_t x = 0; x < m; ++x) st[inst][n++] = C + (int64_t)(2 * s - 1 - i) * m + x; /* S_{2s-1-i} */
            }
            stn[inst] = n;
        }
        C += L;
        off += s;
    }
    if (rc == ORACLE_OK) {
        const int s = sp[upto];
        const int32_t* grp = ranks + off;
        for (int i = 0; i < s; ++i) {
            store_n[i] = stn[grp[i]];
            if (store_pos) {
                if (stn[grp[i]] > pos_stride) { rc = ORACLE_ERR_RANGE; break; }
                memcpy(store_pos + (size_t)i * pos_stride, st[grp[i]], sizeof(int64_t) * (size_t)stn[grp[i]]);
            }
        }
    }
    if (n_moves) *n_moves = nm;
    for (int i = 0; i < n_inst; ++i) free(st[i]);
    free(st); free(stn); free(tmp);
    return rc;
}

/*
 * Decode paged-KV writer.  P:55 (§2.2): PagedAttention manages "the KV cache in block
 * granularity"; prefill instances stream each chunk's KV to the decode
 * instance; decode runs at a larger TP (TP=8 for 8B).  R15 fixes the layout:
 * separate K and V caches per decode TP rank t, each [num_blocks, B, Hkv/tp, D]; KV head h
 * belongs to t = floor(h * tp / Hkv); position p goes to physical block
 * block_table[p / B], row p mod B.
 *
 *   dst[t][ block_table[p/B] ][ p mod B ][ h - t*Hkv/tp ][:] = src[i][h][:]
 *
 * src [n_tok, Hkv, D] of esize-byte elements (a pure byte copy, so bit-exact);
 * pos[i] = global position of src row i.  Returns ORACLE_ERR_RANGE on an out-of-range
 * block-table entry or physical block id.
 */
int oracle_paged_write(const void* src, const int64_t* pos, int64_t n_tok, int Hkv, int D, int esize,
                       int tp, int B, const int32_t* block_table, int64_t n_table, int64_t num_blocks,
                       void* const* dst) {
    if (!src || !pos || !block_table || !dst || tp <= 0 || B <= 0 || Hkv % tp != 0 || esize <= 0)
        return ORACLE_ERR_ARG;
    const int hl = Hkv / tp;
    const size_t row = (size_t)D * esize;
    for (int64_t i = 0; i < n_tok; ++i) {
        const int64_t p = pos[i];
        if (p < 0 || p / B >= n_table) return ORACLE_ERR_RANGE;
        const int64_t blk = block_table[p / B];
        if (blk < 0 || blk >= num_blocks) return ORACLE_ERR_RANGE;
        for (int h = 0; h < Hkv; ++h) {
            const int t = (int)((int64_t)h * tp / Hkv);
            const int hloc = h - t * hl;
            char* d = (char*)dst[t] + (((size_t)blk * B + (size_t)(p % B)) * hl + hloc) * row;
            const char* sp = (const char*)src + ((size_t)i * Hkv + h) * row;
            memcpy(d, sp, row);
        }
    }
    return ORACLE_OK;
}

/*
 * n-way log-sum-exp merge of partial attention results (R3; the paper never writes it,
 * ring attention [20] and FlashAttention [7] imply it).  For each row t and
 * head h, with a_i = lse_i[h, t]:
 *     M   = max_i a_i
 *     lse = M + ln sum_i exp(a_i - M)
 *     O   = sum_i exp(a_i - M) * O_i / sum_i exp(a_i - M)
 * All inputs -inf: O = 0, lse = -inf (never NaN); a -inf part contributes nothing.
 * o_parts[i] [T, H, D], lse_parts[i] [H, T]; out [T, H, D], lse [H, T]; double.
 */
int oracle_lse_merge(int n, const double* const* o_parts, const double* const* lse_parts,
                     int64_t T, int H, int D, double* out, double* lse) {
    if (n <= 0 || !o_parts || !lse_parts || !out || !lse) return ORACLE_ERR_ARG;
    for (int64_t t = 0; t < T; ++t) {
        for (int h = 0; h < H; ++h) {
            double M = -INFINITY;
            for (int i = 0; i < n; ++i) {
                const double a = lse_parts[i][(size_t)h * T + t];
                if (a > M) M = a;
            }
            double* o = out + ((size_t)t * H + h) * D;
            for (int d = 0; d < D; ++d) o[d] = 0.0;
            if (M == -INFINITY) { lse[(size_t)h * T + t] = -INFINITY; continue; }
            double den = 0.0;
            for (int i = 0; i < n; ++i) {
                const double a = lse_parts[i][(size_t)h * T + t];
                if (a == -INFINITY) continue;
                const double w = exp(a - M);
                den += w;
                const double* oi = o_parts[i] + ((size_t)t * H + h) * D;
                for (int d = 0; d < D; ++d) o[d] += w * oi[d];
            }
            for (int d = 0; d < D; ++d) o[d] /= den;
            lse[(size_t)h * T + t] = M + log(den);
        }
    }
    return ORACLE_OK;
}
