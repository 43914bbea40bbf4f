/*
 * cdsp.h — C ABI of the B200-native CDSP chunked-prefill ring-attention library
 * (libcdsp.so, sm_100a).
 *
 * The method: Tetris' Chunkwise Dynamic Sequence Parallelism (arXiv 2511.06247,
 * /root/reference/PAPER.md, cited "P:<line>").  One prompt chunk's causal attention is
 * sharded over an SP group of s in {1,2,4,8} GPUs with the zigzag partition; each
 * rank attends its query shard to all historical KV (prior chunks, re-balanced onto the
 * current group) and to the current chunk's KV, which circulates around the ring
 * (P:59); partial results are combined by log-sum-exp merge; the finished KV is scattered
 * into the decode instance's paged cache.
 *
 * Conventions for every call
 *  - All tensors are caller-owned, contiguous, row-major [T, H, D] (D fastest) device
 *    memory (cdsp_tensor), unless stated otherwise.  The library never frees caller memory.
 *  - Every call validates its arguments on the host BEFORE enqueueing anything: on a
 *    non-OK status nothing was launched.  cdsp_last_error() then returns a thread-local
 *    message.
 *  - Device work is asynchronous and stream-ordered after prior work on `cuda_stream`
 *    (a cudaStream_t; NULL = legacy default stream).  Asynchronous failures surface as
 *    CDSP_ERR_CUDA / CDSP_ERR_COMM on a later call (or cdsp_comm_check()).
 *  - Collective calls (cdsp_prefill_chunk, cdsp_kv_transfer_to_decode) must be made by
 *    every rank of the chunk's group with identical plan and chunk index (NCCL-like).
 *
 * Readings of the paper this interface fixes ("R<n>"):
 *  R1 softmax scale is a parameter (default 1/sqrt(D)); R2 LSE is the natural log, fp32,
 *  layout [H, T]; R3 merge formula; R4 key j = t is visible; R5 zigzag on chunk-local
 *  indices, masks on global positions; R6 L % 2s == 0; R8 balancing pairing; R9 group
 *  nesting; R14 GQA kv head = floor(h / (Hq/Hkv)); R15 paged layout; R16 empty rows
 *  give lse = -inf, O = 0.
 */
#ifndef CDSP_H_
#define CDSP_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define CDSP_API __attribute__((visibility("default")))
#else
#define CDSP_API
#endif

#define CDSP_ABI_VERSION 5
#define CDSP_IPC_HANDLE_BYTES 64   /* one cudaIpcMemHandle_t */
#define CDSP_MAX_SP 8

typedef enum {
    CDSP_OK = 0,
    CDSP_ERR_INVALID = 1,      /* NULL pointer, bad enum, misuse of a handle */
    CDSP_ERR_SHAPE = 2,        /* inconsistent T/H/D, D not in {64,128}, Hq % Hkv != 0, L % 2s != 0 */
    CDSP_ERR_DTYPE = 3,        /* dtype mismatch between q, k, v, out, store */
    CDSP_ERR_PLAN = 4,         /* illegal plan (R9) or caller not in the chunk's group */
    CDSP_ERR_CAPACITY = 5,     /* store / block table / work buffer too small */
    CDSP_ERR_CUDA = 6,         /* a CUDA runtime/driver call failed */
    CDSP_ERR_COMM = 7,         /* peer barrier timed out / IPC failure */
    CDSP_ERR_UNSUPPORTED = 8   /* e.g. decode tp > Hkv (KV-head replication undefined) */
} cdsp_status;

typedef enum { CDSP_F32 = 0, CDSP_BF16 = 1 } cdsp_dtype;

/* How a chunk's tokens are interleaved over its group ("striped/zigzag"; R5, R20):
 * ZIGZAG: 2s shards S_j = [j m, (j+1) m), ring rank i holds S_i then S_{2s-1-i};
 * STRIPED ("evenly-spaced stripes ... round-robin"): token t -> ring rank t mod s,
 * shard row t / s. */
typedef enum { CDSP_ZIGZAG = 0, CDSP_STRIPED = 1 } cdsp_interleave;

/* A contiguous device tensor [T, H, D]; element type `dtype`. */
typedef struct {
    void* ptr;
    int32_t dtype;      /* cdsp_dtype */
    int64_t T, H, D;
} cdsp_tensor;

/* One chunk of the CDSP plan A = [a_0 .. a_{l-1}], a_i = (token count, instance group)
 * (Alg. 1; D1).  ranks[0..sp) is the group's RING ORDER, as instance (world)
 * ranks.  R9: sp in {1,2,4,8}, non-decreasing over chunks, sp_c / sp_{c-1} integral, the
 * previous chunk's ranks[] a prefix of this one's ("each chunk's instance group
 * must include all instances involved in preceding chunks"), ranks distinct, len % (2 sp) == 0. */
typedef struct {
    int64_t len;
    int32_t sp;
    int32_t interleave;     /* cdsp_interleave (0 = zigzag) */
    const int32_t* ranks;   /* host memory */
} cdsp_chunk;

typedef struct {
    int32_t n_chunks;
    const cdsp_chunk* chunks;   /* host memory */
} cdsp_plan;

/* A cache-balancing transfer: ring rank `src` sends store rows
 * [src_off, src_off + n_tok) to ring rank `dst` (ring ranks of the chunk's group). */
typedef struct {
    int32_t src, dst;
    int64_t src_off, n_tok;
} cdsp_move;

/* ---------------------------------------------------------------------------------
 * Communicator: one per process per GPU ("instance").  It owns the instance's KV store
 * (history of the current request, in memory its peers can read over NVLink), one ring
 * receive slot per ring step, the optional fp32 merge accumulators (cdsp_comm_reserve), an
 * internal comm stream, events, arrival flags and the peer barrier flags.
 * ------------------------------------------------------------------------------- */
typedef struct cdsp_comm_s* cdsp_comm;

/* Create the communicator of instance `rank` of `world` on CUDA device `device`.
 * store_cap_tokens: capacity (tokens) of this instance's KV store and of each ring
 * receive slot; must cover the largest (history + shard) any chunk of any plan will
 * hold on one rank.  Hkv, D, dtype: KV geometry of every request served.  Allocates
 * 2 * world * store_cap_tokens * Hkv * D * sizeof(dtype) (+ small) bytes of device memory:
 * the K and V store, plus one K and V receive slot per ring step (world - 1 of them; none
 * when world == 1).  The fp32 merge accumulators are NOT allocated here (cdsp_comm_reserve).
 * Errors: CDSP_ERR_INVALID, CDSP_ERR_SHAPE (D not in {64,128}), CDSP_ERR_CUDA. */
CDSP_API cdsp_status cdsp_comm_create(cdsp_comm* out, int32_t rank, int32_t world, int32_t device,
                                      int64_t store_cap_tokens, int32_t Hkv, int32_t D, int32_t dtype);

/* Same with n_layers per-layer KV stores (one per transformer layer; positions shared): the
 * layer-wise prefill (cdsp_prefill_chunk_layer) overlaps each layer's cache balancing with
 * the previous layer ("Cache-Balancing Latency Overlap", Fig. 6-b).  Allocates
 * (2 n_layers + 2 (world - 1)) * store_cap_tokens * Hkv * D * sizeof(dtype) (+ small) bytes. */
CDSP_API cdsp_status cdsp_comm_create_layers(cdsp_comm* out, int32_t rank, int32_t world, int32_t device,
                                             int64_t store_cap_tokens, int32_t n_layers, int32_t Hkv, int32_t D,
                                             int32_t dtype);

/* Reserve the fp32 merge accumulators (max_q_rows * max_hq * D + max_q_rows * max_hq floats)
 * for rings that run as SEVERAL launches merged through them: f32 rings (one launch per
 * block), bf16 rings whose blocks exceed one launch's KV tile list (4096 tiles of 128 keys at
 * D = 128), and CDSP_RING_STEPWISE.  A bf16 ring that fits one launch needs none (its output
 * stays in tensor memory across the whole ring).  Synchronises the device; grows only;
 * never called by cdsp_prefill_chunk, which fails with CDSP_ERR_CAPACITY instead.
 * Errors: CDSP_ERR_INVALID, CDSP_ERR_CUDA. */
CDSP_API cdsp_status cdsp_comm_reserve(cdsp_comm c, int64_t max_q_rows, int32_t max_hq);

/* Ring options (bits, default 0), for measurement and tests:
 *  CDSP_RING_STEPWISE    one attention launch per ring step, merged through the reserved fp32
 *                        accumulators (the round-1 design; control for the fused ring);
 *  CDSP_RING_CONTROL     no pulls: the receive slots keep the blocks an earlier call with the
 *                        same inputs pulled ("peer blocks pre-staged", SURVEY §8(d)'s control run:
 *                        ring latency minus control latency = the exposed ring time);
 *  CDSP_RING_GATE_FLAGS  gate the fused ring on arrival flags even when a peer shares this GPU
 *                        (default: flags only when every peer is another GPU, else events;
 *                        loopback groups then run their rings one at a time);
 *  CDSP_RING_GATE_EVENTS always wait for a launch's pulls with events. */
#define CDSP_RING_STEPWISE 1
#define CDSP_RING_CONTROL 2
#define CDSP_RING_GATE_FLAGS 4
#define CDSP_RING_GATE_EVENTS 8
CDSP_API cdsp_status cdsp_comm_set_ring_options(cdsp_comm c, int32_t options);

/* Export this instance's shared region as CDSP_IPC_HANDLE_BYTES bytes (host buffer). */
CDSP_API cdsp_status cdsp_comm_ipc_handle(cdsp_comm c, void* handle_out);

/* Multi-process: open every other instance's region.  handles = world * CDSP_IPC_HANDLE_BYTES
 * host bytes, handle i from instance i (entry `rank` is ignored).  All instances must use
 * the same world / store_cap_tokens / n_layers / Hkv / D / dtype: each region carries a
 * geometry header, and a peer whose header differs is refused with CDSP_ERR_COMM (nothing
 * is mapped into the peer's store at a wrong offset).  Peers on another GPU (by UUID) are
 * marked remote: the fused ring then gates on arrival flags instead of events.
 * Errors: CDSP_ERR_COMM, CDSP_ERR_CUDA. */
CDSP_API cdsp_status cdsp_comm_connect(cdsp_comm c, const void* handles);

/* Loopback: `world` communicators created in THIS process on ONE device (comms[i] has
 * rank i) are linked into a group.  cdsp_prefill_chunk then acts as a deferred collective
 * (like an NCCL group call): each ring rank's call is validated and recorded, and the call
 * that completes the chunk's group enqueues every rank's work on the ranks' own streams,
 * ordered by CUDA events (no device-side spinning).  One host thread issues all calls. */
CDSP_API cdsp_status cdsp_comm_connect_local(cdsp_comm* comms, int32_t world);

/* Poll for asynchronous errors (peer-barrier timeout -> CDSP_ERR_COMM).  Does not block. */
CDSP_API cdsp_status cdsp_comm_check(cdsp_comm c);

/* Optional live timing of the block-attention launches this communicator issues inside
 * cdsp_prefill_chunk: with enable != 0, a CUDA event pair brackets each launch on the
 * caller's stream (up to 8192 pairs).  _read synchronises on the last event and returns
 * the summed kernel time (ms) and launch count since the last read, then resets. */
CDSP_API cdsp_status cdsp_comm_profile(cdsp_comm c, int32_t enable);
CDSP_API cdsp_status cdsp_comm_profile_read(cdsp_comm c, double* attn_ms, int32_t* n_launches);

/* Ring profile of the same window (SURVEY §8(d) "ring hidden"): over the ring pulls this
 * communicator issued while profiling (up to 4096), *copy_ms = summed pull durations on the
 * comm stream, *bytes = K+V bytes pulled, *n_pulls = their count, and *exposed_ms = summed
 * time the compute stream had to wait for them: for the pull feeding ring step k,
 * max(0, pull end - end of step k-1's attention).  0 = the ring is fully hidden.  Call before
 * issuing more work (it reads the attention events cdsp_comm_profile_read also reads, in
 * either order); synchronises on them and resets the ring records. */
CDSP_API cdsp_status cdsp_comm_profile_ring(cdsp_comm c, double* copy_ms, double* exposed_ms, int64_t* bytes,
                                            int32_t* n_pulls);

/* Destroy (synchronises the device first).  Peers must be done with this instance. */
CDSP_API cdsp_status cdsp_comm_destroy(cdsp_comm c);

/* Per-instance KV store (D4): the balanced history of the current request followed,
 * after each chunk, by that chunk's zigzag shard.  A VIEW of comm-owned memory:
 * k, v [cap, Hkv, D]; pos int32 [cap] global positions; rows [0, n) valid. */
typedef struct {
    cdsp_tensor k, v;
    int32_t* pos;        /* device */
    int64_t n, cap;
} cdsp_kvstore;

CDSP_API cdsp_status cdsp_kvstore_get(cdsp_comm c, cdsp_kvstore* out);               /* layer 0 */
CDSP_API cdsp_status cdsp_kvstore_get_layer(cdsp_comm c, int32_t layer, cdsp_kvstore* out);

/* Start a new request on this instance: its stores (all layers) become empty (host-side; stream-ordered
 * uses of the old content must be complete or on `cuda_stream`, which this call joins). */
CDSP_API cdsp_status cdsp_kvstore_reset(cdsp_comm c, void* cuda_stream);

/* The SP group executing one chunk: communicator of the calling instance + plan + chunk. */
typedef struct {
    cdsp_comm comm;
    const cdsp_plan* plan;
    int32_t chunk;
} cdsp_sp_group;

/* ---------------------------------------------------------------------------------
 * The four calls of the hot path
 * ------------------------------------------------------------------------------- */

/* Host-only and pure: the store capacity (rows per instance) `plan` needs, i.e. the
 * largest history + shard any ring rank holds over the plan (R8).  Errors: as
 * cdsp_plan_partition. */
CDSP_API cdsp_status cdsp_plan_capacity(const cdsp_plan* plan, int64_t* rows);

/* Host-only and pure.  For chunk c of `plan` (L = len, s = sp, m = L / 2s, C = tokens of
 * earlier chunks) writes (NULL outputs are skipped):
 *   tok_rank[L], tok_slot[L]: chunk-local token t is row tok_slot[t] of ring rank
 *       tok_rank[t]'s shard; zigzag: shard S_j = [j m, (j+1) m) belongs to ring rank
 *       j (j < s) or 2s-1-j, and rank i's shard is S_i followed by S_{2s-1-i}; striped
 *       chunks (R20): tok_rank[t] = t mod s, tok_slot[t] = t / s;
 *   rank_pos[s * 2m]: global position (C + local) of each shard row, rank-major;
 *   moves[<= CDSP_MAX_SP], *n_moves: the balancing transfers executed before chunk c (R8).
 * Errors: CDSP_ERR_INVALID, CDSP_ERR_PLAN. */
CDSP_API cdsp_status cdsp_plan_partition(const cdsp_plan* plan, int32_t c, int32_t* tok_rank,
                                         int32_t* tok_slot, int64_t* rank_pos, cdsp_move* moves,
                                         int32_t* n_moves);

/* Collective over plan->chunks[chunk].ranks.  The calling instance is ring rank r.
 *   q [2m, Hq, D], k/v [2m, Hkv, D]: this rank's shard of the chunk (zigzag: S_r then
 *     S_{2s-1-r}; striped: tokens r, r + s, r + 2s, ...), post-projection ("each instance first calculates its local tokens'
 *     query, key, value"), dtype bf16 or f32 (all equal, = store dtype).
 *   prev_kv: this instance's store view (cdsp_kvstore_get).  Before the chunk, history is
 *     re-balanced from the previous group (R8); afterwards k/v are appended and
 *     prev_kv->n is updated.  prev_kv->n must match the plan (store of chunk `chunk`).
 *   softmax_scale: sigma of s_tj = sigma <q_t, k_j> (R1); <= 0 selects 1/sqrt(D).
 *   out [2m, Hq, D] (dtype of q): exact causal attention of the shard's queries over every
 *     earlier token of the request (history + chunk), RNE-rounded on the final write (R13).
 *   lse: fp32 [Hq, 2m] device, natural log (R2); may be NULL.
 * Errors: CDSP_ERR_INVALID/SHAPE/DTYPE/PLAN/CAPACITY (host validation), CDSP_ERR_CUDA. */
CDSP_API cdsp_status cdsp_prefill_chunk(const cdsp_tensor* q, const cdsp_tensor* k, const cdsp_tensor* v,
                                        cdsp_kvstore* prev_kv, const cdsp_sp_group* sp_group,
                                        float softmax_scale, cdsp_tensor* out, float* lse,
                                        void* cuda_stream);

/* cdsp_prefill_chunk on layer `layer`'s store (0 <= layer < n_layers; prev_kv from
 * cdsp_kvstore_get_layer).  A chunk is processed layer by layer: every rank of the group calls
 * layers 0, 1, ... in order (the caller's per-layer work, e.g. the FC layers, goes between the
 * calls on the same stream).  When the chunk re-balances history (its group grew), layer 0
 * balances inline; right after layer l's ring is enqueued, a new rank issues layer l+1's
 * balancing pulls on its communicator stream, so they run under the rest of layer l and the
 * caller's FC work (Fig. 6-b); layer l+1 then only waits for them.  Old ranks
 * overwrite a moved part only after its puller acknowledged the pull.  Result semantics per
 * layer are exactly cdsp_prefill_chunk's. */
CDSP_API cdsp_status cdsp_prefill_chunk_layer(const cdsp_tensor* q, const cdsp_tensor* k, const cdsp_tensor* v,
                                              cdsp_kvstore* prev_kv, const cdsp_sp_group* sp_group,
                                              int32_t layer, float softmax_scale, cdsp_tensor* out, float* lse,
                                              void* cuda_stream);

/* n >= 1 partial attention results over disjoint key sets -> their combination (R3):
 *   M = max_i lse_i; lse = M + ln sum_i e^{lse_i - M}; O = sum_i e^{lse_i - M} O_i / sum_i e^{lse_i - M}.
 * o_parts[i]: fp32 [T, H, D]; lse_parts[i]: fp32 [H, T] device (rows may be -inf);
 * out [T, H, D] fp32 or bf16 (RNE); lse fp32 [H, T] (may be NULL).  All -inf: O = 0,
 * lse = -inf.  n <= 16.  Errors: CDSP_ERR_INVALID/SHAPE/DTYPE. */
CDSP_API cdsp_status cdsp_lse_merge(int32_t n, const cdsp_tensor* const* o_parts,
                                    const float* const* lse_parts, cdsp_tensor* out, float* lse,
                                    void* cuda_stream);

/* Decode paged-KV destination (R15).  Decode TP rank t (0 <= t < tp) owns KV heads
 * [t Hkv/tp, (t+1) Hkv/tp); its K and V caches are each [num_blocks, block_size, Hkv/tp, D]
 * (dtype of k) at k_cache[t] / v_cache[t] — pointers valid in the caller's address space
 * (local, or peer memory mapped by the caller).  block_table: device int32
 * [n_table], logical block -> physical block; position p lives at
 * (block_table[p / block_size], p mod block_size). */
typedef struct {
    int32_t tp, block_size;
    int64_t num_blocks;
    void* const* k_cache;         /* host array of tp device pointers */
    void* const* v_cache;         /* host array of tp device pointers */
    const int32_t* block_table;   /* device */
    int64_t n_table;
} cdsp_decode_target;

/* Collective-free per-rank scatter of this rank's shard of chunk `chunk` (k, v as passed
 * to cdsp_prefill_chunk) into the decode caches (chunk KV "streamed" to the
 * decode instance).  Bit-exact byte copy.  Requires Hkv % tp == 0 (else
 * CDSP_ERR_UNSUPPORTED) and n_table * block_size > every position (else
 * CDSP_ERR_CAPACITY); block_table entries outside [0, num_blocks) are skipped and counted
 * (see cdsp_kv_transfer_errors). */
CDSP_API cdsp_status cdsp_kv_transfer_to_decode(const cdsp_tensor* k, const cdsp_tensor* v,
                                                const cdsp_sp_group* sp_group,
                                                const cdsp_decode_target* dst, void* cuda_stream);

/* cdsp_prefill_chunk and cdsp_kv_transfer_to_decode of the same k / v in one call (P:135,
 * each chunk's KV is streamed to the decode instance as the chunk is prefilled): the
 * same results, the same decode caches bit for bit and the same error count
 * (cdsp_kv_transfer_errors) as the two calls on cuda_stream.  The attention is enqueued first;
 * the scatter runs on the communicator's own transfer stream (it only reads k / v), filling SMs
 * as the attention's persistent grid frees them, and cuda_stream waits for both.  (Storing
 * each KV tile from the attention's shared-memory stages inside the attention launch was
 * measured slower: DESIGN §6.1.)  Errors: those of the two calls. */
CDSP_API cdsp_status cdsp_prefill_chunk_transfer(const cdsp_tensor* q, const cdsp_tensor* k, const cdsp_tensor* v,
                                                 cdsp_kvstore* prev_kv, const cdsp_sp_group* sp_group,
                                                 float softmax_scale, cdsp_tensor* out, float* lse,
                                                 const cdsp_decode_target* dst, void* cuda_stream);

/* ---------------------------------------------------------------------------------
 * CDSP prefill scheduler (§5.1).  Host-only, pure.
 * ------------------------------------------------------------------------------- */

/* Eq. (1): T_s(R) = a + b L + c (C L) + d L^2 for a chunk of L tokens with C
 * historical tokens at SP size s (a: constant, b: FC layers, c: attention to history,
 * d: attention within the chunk), in any time unit. */
typedef struct {
    double a, b, c, d;
} cdsp_latency_model;

/* Least-squares fit of Eq. (1) to n >= 4 measured (C[i], L[i], T[i]).
 * Errors: CDSP_ERR_INVALID (NULL, too few or rank-deficient samples). */
CDSP_API cdsp_status cdsp_fit_latency_model(int32_t n, const double* C, const double* L, const double* T,
                                            cdsp_latency_model* out);

#define CDSP_MAX_CHUNKS 8
/* A scheduled plan: chunk c has len[c] tokens on the sp[c] instances ranks[c][0..sp) (ring
 * order, nested: chunk c's list starts with chunk c-1's, R9) — the plan A of Alg. 1, ready
 * for cdsp_plan (zigzag chunks); ttft = its Eq. (1) time to first token. */
typedef struct {
    int32_t n_chunks;
    int64_t len[CDSP_MAX_CHUNKS];
    int32_t sp[CDSP_MAX_CHUNKS];
    int32_t ranks[CDSP_MAX_CHUNKS][CDSP_MAX_SP];
    double ttft;
} cdsp_schedule;

/* Algorithm 1 (with Alg. 2 single-chunk scheduling, the GetGroup extension of P:269,
 * Alg. 3 chunk plan solving and the queue update Eq. (2); readings R21-R27) for a new
 * request of L tokens:
 *   queue[n_instances]: each prefill instance's queuing latency T_i (>= 0; model time unit);
 *     instance i lives on node i / node_size;
 *   sizes[n_sizes] (subset of {1,2,4,8}) with models[n_sizes] their Eq. (1) coefficients;
 *   improvement_rate in [0, 1): a larger SP size is taken only if it cuts the estimated TTFT
 *     by more than this fraction (Alg. 2 line 13);
 *   granule: chunk lengths are multiples of it (a multiple of 2 max(sizes), R6/R25); L must be.
 * Errors: CDSP_ERR_INVALID, CDSP_ERR_SHAPE, CDSP_ERR_PLAN (no size fits the pool). */
CDSP_API cdsp_status cdsp_schedule_prefill(int64_t L, int32_t n_instances, const double* queue, int32_t node_size,
                                           int32_t n_sizes, const int32_t* sizes, const cdsp_latency_model* models,
                                           double improvement_rate, int64_t granule, cdsp_schedule* out);

/* ---------------------------------------------------------------------------------
 * Decode consumer of the transferred cache
 * ------------------------------------------------------------------------------- */

/* Workspace bytes cdsp_decode_attention needs for hq_local query heads and hkv_local KV
 * heads of head dim D (independent of the context length).  Errors: CDSP_ERR_SHAPE. */
CDSP_API cdsp_status cdsp_decode_workspace_bytes(int32_t hq_local, int32_t hkv_local, int32_t D, size_t* bytes);

/* One decode step's attention on decode TP rank t, read straight from the paged cache
 * cdsp_kv_transfer_to_decode wrote (§2.2 PagedAttention "block granularity"; §6
 * vLLM components; P:135/P:177 the KV streamed to the decode instance).  The query is the
 * newest token (position n_ctx - 1, its own K/V already in the cache) and sees every cached
 * position 0 .. n_ctx-1 (R4):  o_h = sum_j softmax_j(sigma <q_h, k_{j,kv(h)}>) v_{j,kv(h)}.
 *   q [1, Hq_t, D]: rank t's query heads (global heads [t Hq_t, (t+1) Hq_t)), bf16 or f32 =
 *     the cache dtype; hkv_local = Hkv / tp KV heads in cache->k_cache[t] / v_cache[t]
 *     ([num_blocks, block_size, hkv_local, D]); local head h uses KV head h / (Hq_t/hkv_local) (R14);
 *   softmax_scale: sigma (<= 0: 1/sqrt(D), R1);
 *   out [1, Hq_t, D] (dtype of q, RNE for bf16); lse fp32 [Hq_t] natural log (R2), may be NULL;
 *   workspace: >= cdsp_decode_workspace_bytes, 256-byte aligned device memory, ZERO-FILLED
 *     once before first use (each call leaves it zero-filled again); one call at a time per
 *     workspace.
 * Split-KV flash-decoding in one launch (partials merged in-kernel by R3).  Block-table
 * entries outside [0, num_blocks) contribute no keys.  Errors: CDSP_ERR_INVALID/SHAPE/DTYPE,
 * CDSP_ERR_CAPACITY (n_table * block_size < n_ctx, workspace too small),
 * CDSP_ERR_UNSUPPORTED (Hq_t/hkv_local not in {1,2,4,8}; block_size not a power of two). */
CDSP_API cdsp_status cdsp_decode_attention(const cdsp_tensor* q, const cdsp_decode_target* cache, int32_t t,
                                           int32_t hkv_local, int64_t n_ctx, float softmax_scale,
                                           cdsp_tensor* out, float* lse, void* workspace,
                                           size_t workspace_bytes, void* cuda_stream);

/* The same decode step for a batch of requests in one launch (a decode instance steps every
 * running request at once).  Request b's newest token attends to its positions
 * 0 .. ctx_lens[b]-1 through row b of the block table.
 *   q / out [batch, Hq_t, D] bf16 (request-major); lse fp32 [batch, Hq_t] or NULL;
 *   cache->block_table: device int32 [batch][n_table / batch] (row b = request b's pages);
 *   ctx_lens: HOST int32 [batch] (the decode instance's own record of its requests' lengths),
 *     each >= 1; the splits are sized so that all requests' splits together fill at most one
 *     wave, and laid out back to back on a 1D grid (a request of c tokens gets ceil(c / split)
 *     per KV head); batch <= 1024;
 *   workspace: >= cdsp_decode_workspace_bytes(batch * Hq_t, batch * Hkv_t, D), zero-filled once
 *     (left zero-filled), one call at a time per workspace.
 * Errors: as cdsp_decode_attention; CDSP_ERR_UNSUPPORTED unless bf16 with block_size >= 16 (the
 * TMA kernel); CDSP_ERR_SHAPE if n_table is not a multiple of batch or a length is < 1;
 * CDSP_ERR_CAPACITY if a row covers fewer positions than the longest request, batch > 1024 or
 * batch * Hkv_t > 65535. */
CDSP_API cdsp_status cdsp_decode_attention_batch(const cdsp_tensor* q, const cdsp_decode_target* cache, int32_t t,
                                                 int32_t hkv_local, int32_t batch, const int32_t* ctx_lens,
                                                 float softmax_scale, cdsp_tensor* out, float* lse, void* workspace,
                                                 size_t workspace_bytes, void* cuda_stream);

/* ---------------------------------------------------------------------------------
 * Building blocks, exported for tests and benches (same kernels the path uses)
 * ------------------------------------------------------------------------------- */

/* Segment description of one block-attention launch (one ring step).  With st = pos_stride
 * (0 or 1: contiguous; s for a striped chunk), query row i has global position
 * q_pos0 + i st for i < q_len0, else q_pos1 + (i - q_len0) st.  KV rows [0, kv_hist) are
 * history (always visible); row kv_hist + j has position kv_pos0 + j st for
 * j < kv_len0, else kv_pos1 + (j - kv_len0) st.  Key visible iff its position <= the
 * query's (R4).  Rows >= nq / >= nkv do not exist. */
typedef struct {
    int64_t nq, q_len0, q_pos0, q_pos1;
    int64_t nkv, kv_hist, kv_len0, kv_pos0, kv_pos1;
    int64_t pos_stride;
} cdsp_segments;

/* Merge mode of cdsp_attention_fwd. */
typedef enum {
    CDSP_ATTN_ONLY = 0,   /* final out (+lse) from this block alone                      */
    CDSP_ATTN_FIRST = 1,  /* o_acc/lse_acc := this block                                 */
    CDSP_ATTN_MID = 2,    /* o_acc/lse_acc := merge(acc, this block)                     */
    CDSP_ATTN_LAST = 3    /* out/lse := merge(acc, this block)                           */
} cdsp_attn_mode;
/* OR-ed into the mode of a bf16 MID / LAST launch: launch it as a programmatic dependent of the
 * preceding kernel in the stream.  It may then start while that kernel finishes its last work
 * and touches o_acc / lse_acc / out / lse only after it completed, so the preceding kernel must
 * not write q / k / v (use it to chain FIRST / MID / LAST launches; off by default). */
#define CDSP_ATTN_PDL 0x100

/* One block-attention launch: q [nq, Hq, D]; k, v [nkv, Hkv, D]; o_acc fp32 [nq, Hq, D] and
 * lse_acc fp32 [Hq, nq] (FIRST/MID/LAST); out [nq, Hq, D] dtype of q and lse fp32 [Hq, nq]
 * (ONLY/LAST; lse may be NULL).  bf16 runs the tcgen05/TMEM/TMA kernel, f32 the FFMA kernel.
 * mode may carry CDSP_ATTN_PDL (see there).
 * Errors: CDSP_ERR_INVALID/SHAPE/DTYPE (host validation); CDSP_ERR_CAPACITY when a bf16 block has
 * more than 4096 KV tiles of 128 keys (512K keys per launch; split longer blocks with FIRST /
 * MID / LAST); CDSP_ERR_CUDA. */
CDSP_API cdsp_status cdsp_attention_fwd(const cdsp_tensor* q, const cdsp_tensor* k, const cdsp_tensor* v,
                                        const cdsp_segments* seg, float softmax_scale, int32_t mode,
                                        float* o_acc, float* lse_acc, cdsp_tensor* out, float* lse,
                                        void* cuda_stream);

/* The same over nblk <= 8 KV blocks in ONE launch: the queries attend to the union of the blocks
 * (block b: k[b], v[b] [nkv_b, Hkv, D], described by seg[b]; the query fields q_len0, q_pos0,
 * q_pos1 and pos_stride of every seg[b] must equal seg[0]'s), walked in order with one online
 * softmax per query row — the result is the R3 merge of the per-block attentions without any
 * intermediate partial (a rank's local queries against every block of the ring; P:304
 * "zigzag ring attention for historical tokens").  This is the kernel of a fused ring step
 * sequence.  bf16 only for nblk > 1 (else CDSP_ERR_UNSUPPORTED); all blocks together <= 4096 KV
 * tiles of 128 keys at D = 128 (else CDSP_ERR_CAPACITY).  In CDSP_ATTN_ONLY mode, o_acc / lse_acc
 * (optional, shaped as for FIRST) are scratch: given, the launch may split its heaviest query
 * units over two block ranges and merge the halves (R3) through those rows, so no single unit
 * sets the launch's tail.  Other arguments and errors as cdsp_attention_fwd. */
CDSP_API cdsp_status cdsp_attention_fwd_blocks(const cdsp_tensor* q, int32_t nblk, const cdsp_tensor* const* k,
                                               const cdsp_tensor* const* v, const cdsp_segments* seg,
                                               float softmax_scale, int32_t mode, float* o_acc, float* lse_acc,
                                               cdsp_tensor* out, float* lse, void* cuda_stream);

/* Zigzag gather / scatter: full [L, H, D] <-> ring rank r's shard [2m, H, D]
 * (rows S_r then S_{2s-1-r}).  Bit-exact.  Errors: CDSP_ERR_SHAPE, CDSP_ERR_DTYPE. */
CDSP_API cdsp_status cdsp_zigzag_gather(const cdsp_tensor* full, int32_t s, int32_t r, cdsp_tensor* shard,
                                        void* cuda_stream);
CDSP_API cdsp_status cdsp_zigzag_scatter(const cdsp_tensor* shard, int32_t s, int32_t r, cdsp_tensor* full,
                                         void* cuda_stream);

/* Striped gather / scatter (R20): full [L, H, D] <-> ring rank r's shard [L/s, H, D]
 * (shard row i = full row i s + r).  L % 2s == 0.  Bit-exact. */
CDSP_API cdsp_status cdsp_striped_gather(const cdsp_tensor* full, int32_t s, int32_t r, cdsp_tensor* shard,
                                         void* cuda_stream);
CDSP_API cdsp_status cdsp_striped_scatter(const cdsp_tensor* shard, int32_t s, int32_t r, cdsp_tensor* full,
                                          void* cuda_stream);

/* Device zigzag maps: tok_rank / tok_slot int32 [L] device. */
CDSP_API cdsp_status cdsp_zigzag_map_device(int64_t L, int32_t s, int32_t* tok_rank, int32_t* tok_slot,
                                            void* cuda_stream);

/* Number of block-table entries the last cdsp_kv_transfer_to_decode on this comm found out
 * of range (synchronises `cuda_stream`). */
CDSP_API cdsp_status cdsp_kv_transfer_errors(cdsp_comm c, void* cuda_stream, int64_t* n_bad);

/* Thread-local message of the last non-OK status returned on this thread. */
CDSP_API const char* cdsp_last_error(void);

/* CDSP_ABI_VERSION of the loaded library. */
CDSP_API int32_t cdsp_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* CDSP_H_ */
