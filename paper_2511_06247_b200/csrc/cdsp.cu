// cdsp.cu — the C ABI of libcdsp.so: communicator (peer-readable KV store, ring buffers,
// barriers), the CDSP chunk-prefill orchestration, and the exported building blocks.
//
// Per-call procedure of cdsp_prefill_chunk on ring rank r of chunk c (§4.1, Fig. 5;
// P:59 §2.3 ring attention; §6 "zigzag ring attention for historical tokens"):
//   B1  peer barrier (previous call's peer reads of every store are finished)
//   balancing: a rank new to the group pulls its part of an old rank's store (R8);
//       old ranks keep part 0;                                   then B2 (pulls done)
//   append this rank's k/v shard (and positions) to its store
//   B3  peer barrier (every store holds history + shard)
//   ring, step k = 0..s-1: src = (r - k) mod s (R11: receive from the previous neighbour);
//       the block = src's whole store (history + shard).  Step 0 reads the own store;
//       step k >= 1 pulls src's store over NVLink with the copy engines on the internal comm
//       stream into one of two receive buffers (owner-pull: on NVSwitch every peer is one
//       hop, so the logical ring needs no store-and-forward), overlapped with step k-1's
//       attention; each step's attention LSE-merges into fp32 accumulators in its epilogue
//       and the last step writes the output.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "common.cuh"
#include "internal.h"
#include "plan.h"

namespace cdsp {

static thread_local char g_err[1024] = "";

void set_error(const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}
const char* last_error() { return g_err; }

}  // namespace cdsp

using namespace cdsp;

namespace {
constexpr int kMaxWorld = 8;
constexpr int kMaxHG = 8;  // head groups a gated pull is split into

// Geometry header every communicator writes into its exported region (after the flag
// counters), so cdsp_comm_connect can refuse a peer whose store offsets differ.
struct RegionHeader {
    uint64_t magic;
    int32_t abi, n_layers, Hkv, D, dtype, world;
    int64_t cap;
    uint64_t region_bytes, off_v, off_pos, off_flags;
    unsigned char uuid[16];  // the GPU holding the region
};
constexpr uint64_t kRegionMagic = 0x43445350'52454731ull;  // "CDSPREG1"
constexpr size_t kHeaderOff = 2 * kMaxWorld * sizeof(unsigned long long);  // within the flag page

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

struct PeerView {
    char* k = nullptr;
    char* v = nullptr;
    int32_t* pos = nullptr;
    unsigned long long* flags = nullptr;
};

// Loopback groups (cdsp_comm_connect_local): every instance lives in this process; a chunk's
// cdsp_prefill_chunk calls are collected and issued together, ordered by CUDA events.
struct PendingCall {
    int layer;
    cdsp_tensor q, k, v, out;
    float* lse;
    cdsp_kvstore* prev_kv;
    float scale;
    cudaStream_t st;
    bool set;
};
struct LocalGroup {
    int world = 0;
    cdsp_comm comms[kMaxWorld] = {};
    PendingCall calls[kMaxWorld] = {};
    int pending = 0;
    const cdsp_plan* plan = nullptr;
    int chunk = -1;
    int layer = -1;
    int refs = 0;
};
}  // namespace

struct cdsp_comm_s {
    int rank = 0, world = 1, device = 0;
    int64_t cap = 0;
    int Hkv = 0, D = 0;
    int32_t dtype = CDSP_BF16;
    size_t esize = 2, row_bytes = 0;
    // shared (IPC-exportable) region: K store | V store | positions | barrier flags
    void* region = nullptr;
    size_t region_bytes = 0, off_v = 0, off_pos = 0, off_flags = 0;
    PeerView self;
    PeerView peers[kMaxWorld];
    void* ipc_base[kMaxWorld] = {nullptr};
    bool connected = false;
    // local buffers
    void* recv = nullptr;  // (world - 1) x (K, V) receive slots, cap rows each: slot k-1 takes ring step k's block
    char* recv_k[kMaxWorld] = {};
    char* recv_v[kMaxWorld] = {};
    int n_slots = 0;
    float* o_acc = nullptr;  // fp32 merge accumulators (cdsp_comm_reserve); only multi-launch rings use them
    float* lse_acc = nullptr;
    int64_t acc_rows = 0;
    int32_t acc_hq = 0;
    // ring arrival gating (fused ring over cross-device pulls): gate[k * kMaxHG + hg]
    uint32_t* gate = nullptr;
    uint32_t gate_seq = 0;
    bool peer_remote[kMaxWorld] = {};  // peer j lives on another GPU (copy-engine pulls over NVLink)
    int32_t ring_opts = 0;             // CDSP_RING_* option bits (cdsp_comm_set_ring_options)
    cudaEvent_t ev_pull[kMaxWorld] = {};
    cudaEvent_t ev_ring0 = nullptr;    // timing event at the ring start (profiling)
    unsigned long long sent[kMaxWorld] = {0};
    int* err_host = nullptr;
    int* err_dev = nullptr;
    unsigned long long* bad_count = nullptr;
    cudaStream_t comm_stream = nullptr;
    cudaStream_t xfer_stream = nullptr;  // cdsp_prefill_chunk_transfer's decode-cache scatter
    cudaEvent_t ev_x0 = nullptr, ev_x1 = nullptr;
    cudaEvent_t ev_ready = nullptr, ev_done = nullptr;
    // layers (cdsp_comm_create_layers): one K/V store per layer, positions shared
    int n_layers = 1;
    size_t kv_bytes = 0;                 // bytes of one layer's K (or V) store
    std::vector<int64_t> n_l;            // valid store rows per layer
    std::vector<cudaEvent_t> ev_bal_l;   // per layer: this rank's balancing pulls done
    std::vector<int> prebal;             // per layer: chunk whose balancing was pre-issued, -1 none
    const cdsp_plan* prebal_plan = nullptr;
    unsigned long long ack_expect[kMaxWorld] = {0};  // balancing acks expected from each puller
    // live kernel timing (cdsp_comm_profile)
    bool profiling = false;
    std::vector<cudaEvent_t> prof_ev;  // pairs
    int prof_n = 0;
    // ring profile (cdsp_comm_profile_ring): per pull, events at copy start / copy end (comm
    // stream) and the index of the attention launch the pull must beat (its end event)
    struct RingRec {
        int ev;              // ring_ev[2 ev], ring_ev[2 ev + 1]: pull start / end (comm stream)
        cudaEvent_t from;    // the compute stream waited for this pull from this event on; NULL: no wait
        int64_t bytes;
    };
    std::vector<cudaEvent_t> ring_ev;
    std::vector<RingRec> ring_rec;
    int ring_n = 0;
    // loopback group and its ordering events
    LocalGroup* lg = nullptr;
    cudaEvent_t ev_bal = nullptr, ev_app = nullptr, ev_fin = nullptr;
    bool fin_recorded = false;
};

namespace {

cdsp_status check_tensor(const cdsp_tensor* t, const char* name) {
    CDSP_REQUIRE(t != nullptr, CDSP_ERR_INVALID, "%s is NULL", name);
    CDSP_REQUIRE(dtype_ok(t->dtype), CDSP_ERR_DTYPE, "%s: bad dtype %d", name, t->dtype);
    CDSP_REQUIRE(t->T >= 0 && t->H > 0 && t->D > 0, CDSP_ERR_SHAPE, "%s: bad shape [%lld,%lld,%lld]", name,
                 static_cast<long long>(t->T), static_cast<long long>(t->H), static_cast<long long>(t->D));
    CDSP_REQUIRE(t->T == 0 || t->ptr != nullptr, CDSP_ERR_INVALID, "%s: NULL data", name);
    CDSP_REQUIRE((reinterpret_cast<uintptr_t>(t->ptr) & 15u) == 0, CDSP_ERR_INVALID,
                 "%s: data must be 16-byte aligned", name);
    return CDSP_OK;
}

cdsp_status barrier(cdsp_comm c, const ChunkInfo& ci, cudaStream_t st) {
    BarrierArgs a;
    std::memset(&a, 0, sizeof(a));
    for (int i = 0; i < ci.s; ++i) {
        const int j = ci.ranks[i];
        if (j == c->rank) continue;
        c->sent[j] += 1;
        a.remote[a.n] = c->peers[j].flags + c->rank;
        a.local[a.n] = c->self.flags + j;
        a.target[a.n] = c->sent[j];
        ++a.n;
    }
    a.err = c->err_dev;
    return launch_peer_barrier(a, st);
}

// One block-attention launch over a.nblk KV blocks (bf16: tcgen05 kernel, f32: FFMA kernel),
// bracketed by a CUDA event pair when the communicator is profiling.
cdsp_status run_attention(const AttnArgs& a, cudaStream_t st) {
    return a.dtype == CDSP_BF16 ? launch_attention_tc(a, st) : launch_attention_simt(a, st);
}
cdsp_status run_attention_timed(cdsp_comm c, const AttnArgs& a, cudaStream_t st) {
    const bool rec = c->profiling && c->prof_n * 2 + 1 < static_cast<int>(c->prof_ev.size());
    if (rec) CDSP_CUDA(cudaEventRecord(c->prof_ev[2 * c->prof_n], st));
    CDSP_CHECK_STATUS(run_attention(a, st));
    if (rec) {
        CDSP_CUDA(cudaEventRecord(c->prof_ev[2 * c->prof_n + 1], st));
        ++c->prof_n;
    }
    return CDSP_OK;
}
AttnArgs attn_args(cdsp_comm c, const void* q, int Hq, float scale, int mode, void* out, float* lse) {
    AttnArgs a;
    a.q = q;
    a.dtype = c->dtype;
    a.Hq = Hq;
    a.Hkv = c->Hkv;
    a.D = c->D;
    a.scale = scale;
    a.mode = mode;
    a.o_acc = c->o_acc;
    a.lse_acc = c->lse_acc;
    a.out = out;
    a.lse = lse;
    return a;
}

// Segments of ring rank r's query shard against src's block (history + src's shard).
cdsp_segments segments_for(const ChunkInfo& ci, int r, int src) {
    cdsp_segments sgm;
    sgm.nq = 2 * ci.m;
    sgm.q_len0 = ci.m;
    sgm.q_pos0 = shard_pos0(ci, r);
    sgm.q_pos1 = shard_pos1(ci, r);
    sgm.nkv = ci.hist[src] + 2 * ci.m;
    sgm.kv_hist = ci.hist[src];
    sgm.kv_len0 = ci.m;
    sgm.kv_pos0 = shard_pos0(ci, src);
    sgm.kv_pos1 = shard_pos1(ci, src);
    sgm.pos_stride = shard_stride(ci);
    return sgm;
}

// Per-layer store views (the layers of one instance share geometry and the position array).
inline char* layer_k(cdsp_comm c, const PeerView& pv, int layer) { return pv.k + layer * c->kv_bytes; }
inline char* layer_v(cdsp_comm c, const PeerView& pv, int layer) { return pv.v + layer * c->kv_bytes; }
inline bool balancing(const ChunkInfo& ci) { return ci.s_prev > 0 && ci.s > ci.s_prev; }

// Cache balancing (R8) of one layer's store: a ring rank new to the group pulls its part
// of an old rank's store (copy engines, NVLink when the peer is another GPU); positions move
// with layer 0.  Multi-process: each pull is acknowledged to its source (a system-scope
// counter in the source's flag page) so the source may overwrite that part afterwards;
// loopback (g != NULL) orders the source by the puller's event instead.
cdsp_status phase_balance_pull(cdsp_comm c, const ChunkInfo& ci, int r, int layer, cudaStream_t st, bool ack) {
    BarrierArgs a;
    std::memset(&a, 0, sizeof(a));
    for (int i = 0; i < ci.n_moves; ++i) {
        const cdsp_move& mv = ci.moves[i];
        if (mv.dst != r || mv.n_tok == 0) continue;
        const PeerView& src = c->peers[ci.ranks[mv.src]];
        CDSP_CUDA(cudaMemcpyAsync(layer_k(c, c->self, layer), layer_k(c, src, layer) + mv.src_off * c->row_bytes,
                                  mv.n_tok * c->row_bytes, cudaMemcpyDeviceToDevice, st));
        CDSP_CUDA(cudaMemcpyAsync(layer_v(c, c->self, layer), layer_v(c, src, layer) + mv.src_off * c->row_bytes,
                                  mv.n_tok * c->row_bytes, cudaMemcpyDeviceToDevice, st));
        if (layer == 0)
            CDSP_CUDA(cudaMemcpyAsync(c->self.pos, src.pos + mv.src_off, mv.n_tok * sizeof(int32_t),
                                      cudaMemcpyDeviceToDevice, st));
        if (ack) {  // signal only: the source's ack slot for this instance
            a.remote[a.n] = src.flags + kMaxWorld + c->rank;
            a.local[a.n] = c->self.flags + kMaxWorld + c->rank;
            a.target[a.n] = 0;
            ++a.n;
        }
    }
    if (a.n > 0) {
        a.err = c->err_dev;
        CDSP_CHECK_STATUS(launch_peer_barrier(a, st));
    }
    return CDSP_OK;
}

// Multi-process source side: wait until every puller of this rank acknowledged its pull of
// this layer (cumulative counters, so no reset is ever needed).
cdsp_status phase_balance_wait(cdsp_comm c, const ChunkInfo& ci, int r, cudaStream_t st) {
    BarrierArgs a;
    std::memset(&a, 0, sizeof(a));
    for (int i = 0; i < ci.n_moves; ++i) {
        const cdsp_move& mv = ci.moves[i];
        if (mv.src != r || mv.n_tok == 0) continue;
        const int j = ci.ranks[mv.dst];
        c->ack_expect[j] += 1;
        a.remote[a.n] = nullptr;  // wait only
        a.local[a.n] = c->self.flags + kMaxWorld + j;
        a.target[a.n] = c->ack_expect[j];
        ++a.n;
    }
    if (a.n > 0) {
        a.err = c->err_dev;
        CDSP_CHECK_STATUS(launch_peer_barrier(a, st));
    }
    return CDSP_OK;
}

// Append this rank's shard (k, v and global positions) after its balanced history.
cdsp_status phase_append(cdsp_comm c, const ChunkInfo& ci, int r, int layer, const cdsp_tensor* k,
                         const cdsp_tensor* v, cudaStream_t st) {
    int64_t& n = c->n_l[layer];
    n = ci.hist[r];
    AppendArgs a;
    a.k_src = k->ptr;
    a.v_src = v->ptr;
    a.k_dst = layer_k(c, c->self, layer) + n * c->row_bytes;
    a.v_dst = layer_v(c, c->self, layer) + n * c->row_bytes;
    a.pos_dst = c->self.pos + n;
    a.n_rows = 2 * ci.m;
    a.row_bytes = static_cast<int64_t>(c->row_bytes);
    a.len0 = ci.m;
    a.pos0 = shard_pos0(ci, r);
    a.pos1 = shard_pos1(ci, r);
    a.pos_stride = shard_stride(ci);
    CDSP_CHECK_STATUS(launch_store_append(a, st));
    n += 2 * ci.m;
    return CDSP_OK;
}

// Layer-wise balancing overlap ("once the ring attention in current layer completes,
// its inter-instance communicator can be reused to perform cache balancing for the next
// layer"): right after layer l's ring is enqueued, a puller issues layer l+1's balancing
// pulls on its comm stream, behind the ring pulls, so they run under the rest of layer l
// (its last ring steps and whatever the caller runs next, e.g. the FC layers).
cdsp_status prebalance_next(cdsp_comm c, const ChunkInfo& ci, int r, int layer, const cdsp_plan* plan, bool ack) {
    const int nl = layer + 1;
    if (!balancing(ci) || nl >= c->n_layers) return CDSP_OK;
    static const bool off = getenv("CDSP_NO_PREBALANCE") != nullptr;  // measurement control only
    if (off) return CDSP_OK;
    CDSP_CHECK_STATUS(phase_balance_pull(c, ci, r, nl, c->comm_stream, ack));
    CDSP_CUDA(cudaEventRecord(c->ev_bal_l[nl], c->comm_stream));
    c->prebal[nl] = ci.c;
    c->prebal_plan = plan;
    return CDSP_OK;
}
inline bool prebalanced(cdsp_comm c, const ChunkInfo& ci, int layer, const cdsp_plan* plan) {
    return c->prebal[layer] == ci.c && c->prebal_plan == plan;
}

// cuStreamWriteValue32 through the runtime's driver entry point (no link-time libcuda): the
// stream front end writes the word after the preceding copies, no SM involved.
typedef CUresult (*WriteValue32Fn)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
WriteValue32Fn write_value_fn() {
    static WriteValue32Fn fn = nullptr;
    static bool tried = false;
    if (!tried) {
        tried = true;
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<WriteValue32Fn>(p);
    }
    return fn;
}

// How ring rank r runs chunk ci's ring: blocks k = 0 .. s-1 (k = 0: its own store; k >= 1: the
// store of src = (r - k) mod s, pulled into receive slot k - 1), walked by launches of
// consecutive blocks.  bf16: one launch walks every block with O resident in TMEM (the fused
// ring), unless the blocks exceed the kernel's tile list (then several launches, merged
// through the fp32 accumulators) or CDSP_RING_STEPWISE is set; f32: one launch per block.
struct RingLaunches {
    int n = 0;
    int first[kMaxWorld + 1] = {};  // launch i covers blocks [first[i], first[i + 1])
    bool fused = false;
};
// A launch's units each walk all of its blocks, and the units in flight (head-major) are at
// different points of that walk: the K / V of one KV head over all the launch's blocks is the
// L2 working set.  Blocks are grouped so that it stays within this budget (the whole ring in one
// launch for the 32K-token chunk at s = 8: 16.8 MB; one launch per block for a 512K chunk).
int64_t ring_l2_budget() {
    static const int64_t mb = getenv("CDSP_RING_L2_MB") ? atoll(getenv("CDSP_RING_L2_MB")) : 32;
    return mb << 20;
}
cdsp_status ring_launches(cdsp_comm c, const ChunkInfo& ci, int r, RingLaunches* out, int Hq) {
    const bool fused = c->dtype == CDSP_BF16 && !(c->ring_opts & CDSP_RING_STEPWISE);
    // the L2 grouping needs the merge accumulators; without them the whole ring is one launch
    const bool acc_ok = c->acc_rows >= 2 * ci.m && c->acc_hq >= Hq;
    const int max_t = c->dtype == CDSP_BF16 ? attention_tc_max_tiles(c->D) : 0;
    const int64_t head_bytes_per_row = 2ll * c->D * static_cast<int64_t>(c->esize);  // K + V of one KV head
    out->n = 0;
    out->fused = fused;
    int64_t acc = 0, acc_bytes = 0;
    for (int k = 0; k < ci.s; ++k) {
        const int src = (r - k + ci.s) % ci.s;
        const int64_t rows = ci.hist[src] + 2 * ci.m;
        const int64_t t = (rows + 127) / 128;
        CDSP_REQUIRE(c->dtype != CDSP_BF16 || t <= max_t, CDSP_ERR_CAPACITY,
                     "ring block of %lld tiles exceeds the %d KV tiles of one launch", static_cast<long long>(t),
                     max_t);
        const int64_t bytes = rows * head_bytes_per_row;
        if (k == 0 || !fused || acc + t > max_t || (acc_ok && acc_bytes + bytes > ring_l2_budget())) {
            out->first[out->n++] = k;
            acc = 0;
            acc_bytes = 0;
        }
        acc += t;
        acc_bytes += bytes;
    }
    out->first[out->n] = ci.s;
    // Pull pacing (flag-gated rings: every peer on another GPU, or CDSP_RING_GATE_FLAGS).  Every
    // unit of one fused launch walks all the blocks, so its first wave of units cannot finish
    // before the last pull has landed: T_fused ~ T_pull + T_compute (1 - 1 / waves).  When the
    // pulls are long against the compute (a short chunk at s = 8), launches of g blocks — each
    // waiting for its own blocks' pulls, merged through the fp32 accumulators, ~4.4% of T_compute
    // per extra launch (s = 8 stepwise vs fused, blocks resident) — finish earlier.  The model's
    // rates: CDSP_RING_LINK_GBS (pull, default 700) and CDSP_RING_TFLOPS (attention, default 1200).
    bool remote_all = true;
    for (int k = 1; k < ci.s; ++k)
        if (!c->peer_remote[ci.ranks[(r - k + ci.s) % ci.s]]) remote_all = false;
    const bool flags = (c->ring_opts & CDSP_RING_GATE_FLAGS) || (remote_all && !(c->ring_opts & CDSP_RING_GATE_EVENTS));
    if (fused && acc_ok && flags && out->n == 1 && ci.s > 2) {
        static const double link = (getenv("CDSP_RING_LINK_GBS") ? atof(getenv("CDSP_RING_LINK_GBS")) : 700.0) * 1e9;
        static const double rate = (getenv("CDSP_RING_TFLOPS") ? atof(getenv("CDSP_RING_TFLOPS")) : 1200.0) * 1e12;
        double arrive[kMaxWorld + 1] = {}, comp[kMaxWorld] = {}, t_c = 0.0;
        for (int k = 0; k < ci.s; ++k) {
            const int src = (r - k + ci.s) % ci.s;
            const double rows = static_cast<double>(ci.hist[src]) + 2.0 * ci.m;
            // visible pairs: history rows fully, the shard's 2m rows about half (causal / zigzag)
            const double pairs = 2.0 * ci.m * (static_cast<double>(ci.hist[src]) + 0.5 * 2.0 * ci.m);
            comp[k] = 4.0 * c->D * Hq * pairs / rate;
            t_c += comp[k];
            arrive[k] = k == 0 ? 0.0 : arrive[k - 1] + 2.0 * rows * static_cast<double>(c->row_bytes) / link;
        }
        int sms = 148;
        if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device) != cudaSuccess || sms < 2) sms = 148;
        const double units = std::ceil(2.0 * ci.m / 256.0) * Hq, waves = std::max(1.0, units / (sms / 2));
        const double t_fused = std::max(arrive[ci.s - 1] + t_c * (1.0 - 1.0 / waves), t_c);
        int best_g = ci.s;
        double best_t = t_fused;
        for (int g = 1; g < ci.s; ++g) {
            double t = 0.0;
            for (int k0 = 0, i = 0; k0 < ci.s; k0 += g, ++i) {
                const int k1 = std::min(ci.s, k0 + g);
                double cl = 0.0;
                for (int k = k0; k < k1; ++k) cl += comp[k];
                t = std::max(t, arrive[k1 - 1]) + cl + (i > 0 ? 0.044 * t_c : 0.0);
            }
            if (t < 0.9 * best_t) {
                best_t = t;
                best_g = g;
            }
        }
        if (best_g < ci.s) {
            out->n = 0;
            for (int k0 = 0; k0 < ci.s; k0 += best_g) out->first[out->n++] = k0;
            out->first[out->n] = ci.s;
        }
    }
    return CDSP_OK;
}

// The ring (R10, R11): ring step k's block is src = (r - k) mod s's whole store
// (history + shard).  Every pull is issued up front on the comm stream (copy engines; over
// NVLink when the peer is another GPU) into its own receive slot, so the transfers run
// back to back under the attention.  The attention walks the blocks in ring order:
//  * events: a launch starts once the pulls of its blocks landed (same-device peers, where a
//    device-to-device copy may itself need SMs, and multi-launch rings);
//  * arrival flags (fused ring, every peer on another GPU): the launch starts at once on its
//    own block and each producer warp waits for block k's flag (written by the comm stream
//    behind block k's pull, per head group, so the first units' heads arrive first) right
//    before that block's first tile.
// g != NULL (loopback): each pull waits for src's append event.
cdsp_status phase_ring(cdsp_comm c, const ChunkInfo& ci, int r, int layer, const void* q, int Hq, void* out,
                       float* lse, float scale, cudaStream_t st, LocalGroup* g) {
    const int64_t m2 = 2 * ci.m;
    const int s = ci.s;
    RingLaunches rl;
    CDSP_CHECK_STATUS(ring_launches(c, ci, r, &rl, Hq));
    const bool control = (c->ring_opts & CDSP_RING_CONTROL) != 0;
    bool remote_all = true;
    for (int k = 1; k < s; ++k)
        if (!c->peer_remote[ci.ranks[(r - k + s) % s]]) remote_all = false;
    const bool want_flags = (c->ring_opts & CDSP_RING_GATE_FLAGS) ||
                            (remote_all && !(c->ring_opts & CDSP_RING_GATE_EVENTS));
    const bool gating = rl.fused && rl.n == 1 && s > 1 && !control && want_flags && c->gate && write_value_fn();
    // head groups of a gated pull: >= 2 KB per row piece (copy-engine friendly), <= kMaxHG
    int ng = 1;
    if (gating) {
        static const int ng_env = getenv("CDSP_RING_NG") ? atoi(getenv("CDSP_RING_NG")) : 0;
        ng = ng_env > 0 ? ng_env : static_cast<int>(c->row_bytes / 2048);
        if (ng > kMaxHG) ng = kMaxHG;
        if (ng < 1) ng = 1;
        while (c->Hkv % ng != 0) --ng;
    }
    const uint32_t seq = ++c->gate_seq;
    CDSP_CUDA(cudaEventRecord(c->ev_ready, st));  // receive slots are free after st's earlier work
    CDSP_CUDA(cudaStreamWaitEvent(c->comm_stream, c->ev_ready, 0));
    const bool prof = c->profiling && c->ev_ring0 != nullptr;
    if (prof) CDSP_CUDA(cudaEventRecord(c->ev_ring0, st));
    int rec_last[kMaxWorld];  // ring profile record of step k's last pull piece
    for (int k = 0; k < kMaxWorld; ++k) rec_last[k] = -1;
    if (!control) {
        for (int hg = 0; hg < ng; ++hg) {
            for (int k = 1; k < s; ++k) {
                const int src = (r - k + s) % s;
                if (g && hg == 0) CDSP_CUDA(cudaStreamWaitEvent(c->comm_stream, g->comms[ci.ranks[src]]->ev_app, 0));
                const PeerView& pv = c->peers[ci.ranks[src]];
                const int64_t rows = ci.hist[src] + m2;
                const bool rec = prof && c->ring_n < static_cast<int>(c->ring_rec.size());
                if (rec) CDSP_CUDA(cudaEventRecord(c->ring_ev[2 * c->ring_n], c->comm_stream));
                if (ng == 1) {
                    const size_t bytes = static_cast<size_t>(rows) * c->row_bytes;
                    CDSP_CUDA(cudaMemcpyAsync(c->recv_k[k - 1], layer_k(c, pv, layer), bytes, cudaMemcpyDeviceToDevice,
                                              c->comm_stream));
                    CDSP_CUDA(cudaMemcpyAsync(c->recv_v[k - 1], layer_v(c, pv, layer), bytes, cudaMemcpyDeviceToDevice,
                                              c->comm_stream));
                } else {  // head group hg: a 2D copy of its slice of every row
                    const size_t w = c->row_bytes / ng, off = hg * w;
                    CDSP_CUDA(cudaMemcpy2DAsync(c->recv_k[k - 1] + off, c->row_bytes, layer_k(c, pv, layer) + off,
                                                c->row_bytes, w, rows, cudaMemcpyDeviceToDevice, c->comm_stream));
                    CDSP_CUDA(cudaMemcpy2DAsync(c->recv_v[k - 1] + off, c->row_bytes, layer_v(c, pv, layer) + off,
                                                c->row_bytes, w, rows, cudaMemcpyDeviceToDevice, c->comm_stream));
                }
                if (rec) {
                    CDSP_CUDA(cudaEventRecord(c->ring_ev[2 * c->ring_n + 1], c->comm_stream));
                    c->ring_rec[c->ring_n] = {c->ring_n, nullptr,
                                              2 * static_cast<int64_t>(rows) * static_cast<int64_t>(c->row_bytes / ng)};
                    rec_last[k] = c->ring_n++;
                }
                if (gating) {
                    const CUresult e = write_value_fn()(reinterpret_cast<CUstream>(c->comm_stream),
                                                        reinterpret_cast<CUdeviceptr>(c->gate + k * kMaxHG + hg), seq, 0);
                    CDSP_REQUIRE(e == CUDA_SUCCESS, CDSP_ERR_CUDA, "cuStreamWriteValue32 failed (%d)", static_cast<int>(e));
                }
                if (hg == ng - 1) CDSP_CUDA(cudaEventRecord(c->ev_pull[k], c->comm_stream));
            }
        }
    }
    for (int i = 0; i < rl.n; ++i) {
        const int k0 = rl.first[i], k1 = rl.first[i + 1];
        if (!control && !gating && k1 - 1 >= 1) {  // the launch's blocks have landed (the comm stream is in order)
            CDSP_CUDA(cudaStreamWaitEvent(st, c->ev_pull[k1 - 1], 0));
            const int rc = rec_last[k1 - 1];
            if (rc >= 0)  // exposed: from the previous launch's end (or the ring start) to this pull's end
                c->ring_rec[rc].from = i == 0 || c->prof_n == 0 ? c->ev_ring0 : c->prof_ev[2 * (c->prof_n - 1) + 1];
        }
        const int mode = rl.n == 1 ? CDSP_ATTN_ONLY
                                   : (i == 0 ? CDSP_ATTN_FIRST : (i == rl.n - 1 ? CDSP_ATTN_LAST : CDSP_ATTN_MID));
        AttnArgs a = attn_args(c, q, Hq, scale, mode, out, lse);
        a.nblk = k1 - k0;
        a.pdl = i > 0;  // the accumulator is this chain's own
        // one launch: heavy units may be split and merged through the accumulator rows when
        // they are reserved for this shard
        a.split_ok = rl.n == 1 && c->acc_rows >= m2 && c->acc_hq >= Hq;
        if (!a.split_ok && rl.n == 1) a.o_acc = a.lse_acc = nullptr;
        for (int k = k0; k < k1; ++k) {
            const int b = k - k0;
            a.k[b] = k == 0 ? layer_k(c, c->self, layer) : c->recv_k[k - 1];
            a.v[b] = k == 0 ? layer_v(c, c->self, layer) : c->recv_v[k - 1];
            a.seg[b] = segments_for(ci, r, (r - k + s) % s);
        }
        if (gating) {
            a.gate = c->gate;
            a.gate_target = seq;
            a.gate_mask = ((1u << a.nblk) - 1u) & ~1u;  // block 0 is the own store
            a.gate_ng = kMaxHG;
            a.gate_hpg = c->Hkv / ng;
            a.gate_err = c->err_dev;
            if (!remote_all) a.spare_sms = 8;  // forced flags over same-device copies: leave SMs to them
        }
        CDSP_CHECK_STATUS(run_attention_timed(c, a, st));
    }
    CDSP_CUDA(cudaEventRecord(c->ev_done, c->comm_stream));
    CDSP_CUDA(cudaStreamWaitEvent(st, c->ev_done, 0));
    return CDSP_OK;
}

// Loopback execution of one chunk's layer by all its ranks, ordered by events:
//   previous calls finished -> balancing pulls (unless pre-issued by the previous layer) ->
//   (old ranks wait for their pullers) append -> ring (each pull waits for the source's
//   append) -> finish event -> next layer's balancing pulls on the pullers' comm streams.
cdsp_status run_group_local(LocalGroup* g, const ChunkInfo& ci, int layer) {
    auto comm_of = [&](int r) { return g->comms[ci.ranks[r]]; };
    for (int r = 0; r < ci.s; ++r)
        for (int j = 0; j < ci.s; ++j)
            if (comm_of(j)->fin_recorded) CDSP_CUDA(cudaStreamWaitEvent(g->calls[r].st, comm_of(j)->ev_fin, 0));
    if (balancing(ci)) {
        for (int r = 0; r < ci.s; ++r) {
            cdsp_comm c = comm_of(r);
            if (!prebalanced(c, ci, layer, g->plan)) {
                CDSP_CHECK_STATUS(phase_balance_pull(c, ci, r, layer, g->calls[r].st, false));
                CDSP_CUDA(cudaEventRecord(c->ev_bal_l[layer], g->calls[r].st));
            } else {
                CDSP_CUDA(cudaStreamWaitEvent(g->calls[r].st, c->ev_bal_l[layer], 0));
            }
        }
        for (int i = 0; i < ci.n_moves; ++i)  // an old rank overwrites its moved parts only after the pull
            CDSP_CUDA(cudaStreamWaitEvent(g->calls[ci.moves[i].src].st, comm_of(ci.moves[i].dst)->ev_bal_l[layer], 0));
    }
    for (int r = 0; r < ci.s; ++r) {
        PendingCall& pc = g->calls[r];
        CDSP_CHECK_STATUS(phase_append(comm_of(r), ci, r, layer, &pc.k, &pc.v, pc.st));
        CDSP_CUDA(cudaEventRecord(comm_of(r)->ev_app, pc.st));
        pc.prev_kv->n = comm_of(r)->n_l[layer];
    }
    // forced arrival flags on one device (a test of the gating path): the rings run one after
    // another once every append is done, so a spinning persistent grid never starves the
    // append kernels or the same-device copies it waits for (they get the SMs it leaves free)
    const bool serial = (comm_of(0)->ring_opts & CDSP_RING_GATE_FLAGS) != 0;
    for (int r = 0; r < ci.s; ++r) {
        PendingCall& pc = g->calls[r];
        if (serial) {
            for (int j = 0; j < ci.s; ++j) CDSP_CUDA(cudaStreamWaitEvent(pc.st, comm_of(j)->ev_app, 0));
            if (r > 0) CDSP_CUDA(cudaStreamWaitEvent(pc.st, comm_of(r - 1)->ev_fin, 0));
        }
        CDSP_CHECK_STATUS(phase_ring(comm_of(r), ci, r, layer, pc.q.ptr, static_cast<int>(pc.q.H), pc.out.ptr,
                                     pc.lse, pc.scale, pc.st, g));
        if (serial) CDSP_CUDA(cudaEventRecord(comm_of(r)->ev_fin, pc.st));
    }
    for (int r = 0; r < ci.s; ++r) {
        CDSP_CUDA(cudaEventRecord(comm_of(r)->ev_fin, g->calls[r].st));
        comm_of(r)->fin_recorded = true;
    }
    for (int r = 0; r < ci.s; ++r) CDSP_CHECK_STATUS(prebalance_next(comm_of(r), ci, r, layer, g->plan, false));
    return CDSP_OK;
}

}  // namespace

extern "C" {

const char* cdsp_last_error(void) { return cdsp::last_error(); }
int32_t cdsp_abi_version(void) { return CDSP_ABI_VERSION; }

// ------------------------------------------------------------------------------- comm
cdsp_status cdsp_comm_create(cdsp_comm* out, int32_t rank, int32_t world, int32_t device, int64_t store_cap_tokens,
                             int32_t Hkv, int32_t D, int32_t dtype) {
    return cdsp_comm_create_layers(out, rank, world, device, store_cap_tokens, 1, Hkv, D, dtype);
}

cdsp_status cdsp_comm_create_layers(cdsp_comm* out, int32_t rank, int32_t world, int32_t device,
                                    int64_t store_cap_tokens, int32_t n_layers, int32_t Hkv, int32_t D, int32_t dtype) {
    CDSP_REQUIRE(out != nullptr, CDSP_ERR_INVALID, "out is NULL");
    *out = nullptr;
    CDSP_REQUIRE(world >= 1 && world <= kMaxWorld, CDSP_ERR_INVALID, "world %d not in [1,%d]", world, kMaxWorld);
    CDSP_REQUIRE(rank >= 0 && rank < world, CDSP_ERR_INVALID, "rank %d not in [0,%d)", rank, world);
    CDSP_REQUIRE(store_cap_tokens >= 1 && Hkv >= 1, CDSP_ERR_SHAPE, "bad store geometry");
    CDSP_REQUIRE(n_layers >= 1 && n_layers <= 1024, CDSP_ERR_INVALID, "n_layers %d not in [1,1024]", n_layers);
    CDSP_REQUIRE(D == 64 || D == 128, CDSP_ERR_SHAPE, "head dim %d not in {64,128}", D);
    CDSP_REQUIRE(dtype_ok(dtype), CDSP_ERR_DTYPE, "bad dtype %d", dtype);
    CDSP_CUDA(cudaSetDevice(device));
    CDSP_CHECK_STATUS(attention_device_init());  // kernel counters: no allocation on the prefill path
    cdsp_comm c = new cdsp_comm_s();
    c->rank = rank;
    c->world = world;
    c->device = device;
    c->cap = store_cap_tokens;
    c->Hkv = Hkv;
    c->D = D;
    c->dtype = dtype;
    c->esize = dtype_size(dtype);
    c->row_bytes = static_cast<size_t>(Hkv) * D * c->esize;
    const size_t kv_bytes = align_up(static_cast<size_t>(store_cap_tokens) * c->row_bytes, 256);
    c->n_layers = n_layers;
    c->kv_bytes = kv_bytes;
    c->n_l.assign(n_layers, 0);
    c->prebal.assign(n_layers, -1);
    c->ev_bal_l.assign(n_layers, nullptr);
    c->off_v = static_cast<size_t>(n_layers) * kv_bytes;
    c->off_pos = 2 * static_cast<size_t>(n_layers) * kv_bytes;
    c->off_flags = c->off_pos + align_up(static_cast<size_t>(store_cap_tokens) * 4, 256);
    // flag page: [0, 8) peer-barrier counters, [8, 16) balancing-ack counters (per peer), then
    // the geometry header peers check on connect
    c->region_bytes = c->off_flags + align_up(kHeaderOff + sizeof(RegionHeader), 256);
    auto fail = [&](cudaError_t e, const char* what) {
        set_error("%s failed: %s", what, cudaGetErrorString(e));
        cdsp_comm_destroy(c);
        return CDSP_ERR_CUDA;
    };
    cudaError_t e = cudaMalloc(&c->region, c->region_bytes);
    if (e != cudaSuccess) return fail(e, "cudaMalloc(store)");
    e = cudaMemset(c->region, 0, c->region_bytes);
    if (e != cudaSuccess) return fail(e, "cudaMemset(store)");
    char* base = static_cast<char*>(c->region);
    c->self.k = base;
    c->self.v = base + c->off_v;
    c->self.pos = reinterpret_cast<int32_t*>(base + c->off_pos);
    c->self.flags = reinterpret_cast<unsigned long long*>(base + c->off_flags);
    c->peers[rank] = c->self;
    {
        RegionHeader h;
        std::memset(&h, 0, sizeof(h));
        h.magic = kRegionMagic;
        h.abi = CDSP_ABI_VERSION;
        h.n_layers = n_layers;
        h.Hkv = Hkv;
        h.D = D;
        h.dtype = dtype;
        h.world = world;
        h.cap = store_cap_tokens;
        h.region_bytes = c->region_bytes;
        h.off_v = c->off_v;
        h.off_pos = c->off_pos;
        h.off_flags = c->off_flags;
        cudaDeviceProp prop;
        e = cudaGetDeviceProperties(&prop, device);
        if (e != cudaSuccess) return fail(e, "cudaGetDeviceProperties");
        std::memcpy(h.uuid, &prop.uuid, sizeof(h.uuid));
        e = cudaMemcpy(base + c->off_flags + kHeaderOff, &h, sizeof(h), cudaMemcpyHostToDevice);
        if (e != cudaSuccess) return fail(e, "cudaMemcpy(header)");
    }
    // one receive slot (K and V, cap rows each) per ring step k = 1 .. world-1
    c->n_slots = world - 1;
    if (c->n_slots > 0) {
        e = cudaMalloc(&c->recv, 2 * static_cast<size_t>(c->n_slots) * kv_bytes);
        if (e != cudaSuccess) return fail(e, "cudaMalloc(recv)");
        for (int b = 0; b < c->n_slots; ++b) {
            c->recv_k[b] = static_cast<char*>(c->recv) + (2 * b) * kv_bytes;
            c->recv_v[b] = static_cast<char*>(c->recv) + (2 * b + 1) * kv_bytes;
        }
        e = cudaMalloc(reinterpret_cast<void**>(&c->gate), kMaxWorld * kMaxHG * sizeof(uint32_t));
        if (e != cudaSuccess) return fail(e, "cudaMalloc(gate)");
        e = cudaMemset(c->gate, 0, kMaxWorld * kMaxHG * sizeof(uint32_t));
        if (e != cudaSuccess) return fail(e, "cudaMemset(gate)");
    }
    e = cudaHostAlloc(reinterpret_cast<void**>(&c->err_host), sizeof(int), cudaHostAllocMapped);
    if (e != cudaSuccess) return fail(e, "cudaHostAlloc");
    *c->err_host = 0;
    e = cudaHostGetDevicePointer(reinterpret_cast<void**>(&c->err_dev), c->err_host, 0);
    if (e != cudaSuccess) return fail(e, "cudaHostGetDevicePointer");
    e = cudaMalloc(reinterpret_cast<void**>(&c->bad_count), sizeof(unsigned long long));
    if (e != cudaSuccess) return fail(e, "cudaMalloc(bad_count)");
    e = cudaMemset(c->bad_count, 0, sizeof(unsigned long long));
    if (e != cudaSuccess) return fail(e, "cudaMemset");
    e = cudaStreamCreateWithFlags(&c->comm_stream, cudaStreamNonBlocking);
    if (e != cudaSuccess) return fail(e, "cudaStreamCreate");
    e = cudaStreamCreateWithFlags(&c->xfer_stream, cudaStreamNonBlocking);
    if (e != cudaSuccess) return fail(e, "cudaStreamCreate");
    cudaEvent_t* evs[7] = {&c->ev_ready, &c->ev_done, &c->ev_bal, &c->ev_app, &c->ev_fin, &c->ev_x0, &c->ev_x1};
    for (auto* ev : evs) {
        e = cudaEventCreateWithFlags(ev, cudaEventDisableTiming);
        if (e != cudaSuccess) return fail(e, "cudaEventCreate");
    }
    for (auto& ev : c->ev_pull) {
        e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
        if (e != cudaSuccess) return fail(e, "cudaEventCreate");
    }
    for (auto& ev : c->ev_bal_l) {
        e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
        if (e != cudaSuccess) return fail(e, "cudaEventCreate");
    }
    e = cudaDeviceSynchronize();
    if (e != cudaSuccess) return fail(e, "cudaDeviceSynchronize");
    *out = c;
    return CDSP_OK;
}

cdsp_status cdsp_comm_reserve(cdsp_comm c, int64_t max_q_rows, int32_t max_hq) {
    CDSP_REQUIRE(c != nullptr, CDSP_ERR_INVALID, "NULL comm");
    CDSP_REQUIRE(max_q_rows >= 0 && max_hq >= 0, CDSP_ERR_INVALID, "negative reservation");
    if (max_q_rows <= c->acc_rows && max_hq <= c->acc_hq) return CDSP_OK;
    const int64_t rows = max_q_rows > c->acc_rows ? max_q_rows : c->acc_rows;
    const int32_t hq = max_hq > c->acc_hq ? max_hq : c->acc_hq;
    CDSP_CUDA(cudaSetDevice(c->device));
    CDSP_CUDA(cudaDeviceSynchronize());  // no launch may still use the old buffers
    if (c->o_acc) CDSP_CUDA(cudaFree(c->o_acc));
    if (c->lse_acc) CDSP_CUDA(cudaFree(c->lse_acc));
    c->o_acc = nullptr;
    c->lse_acc = nullptr;
    c->acc_rows = 0;
    c->acc_hq = 0;
    CDSP_CUDA(cudaMalloc(reinterpret_cast<void**>(&c->o_acc), static_cast<size_t>(rows) * hq * c->D * sizeof(float)));
    CDSP_CUDA(cudaMalloc(reinterpret_cast<void**>(&c->lse_acc), static_cast<size_t>(rows) * hq * sizeof(float)));
    c->acc_rows = rows;
    c->acc_hq = hq;
    return CDSP_OK;
}

cdsp_status cdsp_comm_set_ring_options(cdsp_comm c, int32_t options) {
    CDSP_REQUIRE(c != nullptr, CDSP_ERR_INVALID, "NULL comm");
    CDSP_REQUIRE((options & ~(CDSP_RING_STEPWISE | CDSP_RING_CONTROL | CDSP_RING_GATE_FLAGS | CDSP_RING_GATE_EVENTS)) == 0,
                 CDSP_ERR_INVALID, "unknown ring option bits 0x%x", options);
    CDSP_REQUIRE(!((options & CDSP_RING_GATE_FLAGS) && (options & CDSP_RING_GATE_EVENTS)), CDSP_ERR_INVALID,
                 "CDSP_RING_GATE_FLAGS and CDSP_RING_GATE_EVENTS exclude each other");
    c->ring_opts = options;
    return CDSP_OK;
}

cdsp_status cdsp_comm_ipc_handle(cdsp_comm c, void* handle_out) {
    CDSP_REQUIRE(c && handle_out, CDSP_ERR_INVALID, "NULL argument");
    static_assert(sizeof(cudaIpcMemHandle_t) == CDSP_IPC_HANDLE_BYTES, "IPC handle size");
    cudaIpcMemHandle_t h;
    CDSP_CUDA(cudaIpcGetMemHandle(&h, c->region));
    std::memcpy(handle_out, &h, sizeof(h));
    return CDSP_OK;
}

cdsp_status cdsp_comm_connect(cdsp_comm c, const void* handles) {
    CDSP_REQUIRE(c && handles, CDSP_ERR_INVALID, "NULL argument");
    CDSP_REQUIRE(!c->connected, CDSP_ERR_INVALID, "communicator already connected");
    CDSP_CUDA(cudaSetDevice(c->device));
    RegionHeader mine;
    CDSP_CUDA(cudaMemcpy(&mine, static_cast<char*>(c->region) + c->off_flags + kHeaderOff, sizeof(mine),
                         cudaMemcpyDeviceToHost));
    const char* hb = static_cast<const char*>(handles);
    for (int j = 0; j < c->world; ++j) {
        if (j == c->rank) continue;
        cudaIpcMemHandle_t h;
        std::memcpy(&h, hb + static_cast<size_t>(j) * CDSP_IPC_HANDLE_BYTES, sizeof(h));
        void* base = nullptr;
        cudaError_t e = cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess);
        CDSP_REQUIRE(e == cudaSuccess, CDSP_ERR_COMM, "cudaIpcOpenMemHandle(peer %d): %s", j, cudaGetErrorString(e));
        c->ipc_base[j] = base;
        char* b = static_cast<char*>(base);
        // the peer's geometry must match this one's: every peer offset below is computed locally
        RegionHeader ph;
        e = cudaMemcpy(&ph, b + c->off_flags + kHeaderOff, sizeof(ph), cudaMemcpyDeviceToHost);
        CDSP_REQUIRE(e == cudaSuccess, CDSP_ERR_COMM, "reading peer %d's header: %s", j, cudaGetErrorString(e));
        CDSP_REQUIRE(ph.magic == kRegionMagic && ph.abi == mine.abi && ph.n_layers == mine.n_layers &&
                         ph.Hkv == mine.Hkv && ph.D == mine.D && ph.dtype == mine.dtype && ph.world == mine.world &&
                         ph.cap == mine.cap && ph.region_bytes == mine.region_bytes && ph.off_v == mine.off_v &&
                         ph.off_pos == mine.off_pos && ph.off_flags == mine.off_flags,
                     CDSP_ERR_COMM,
                     "peer %d's communicator geometry differs (cap %lld/%lld, layers %d/%d, Hkv %d/%d, D %d/%d, "
                     "dtype %d/%d, world %d/%d)",
                     j, static_cast<long long>(ph.cap), static_cast<long long>(mine.cap), ph.n_layers, mine.n_layers,
                     ph.Hkv, mine.Hkv, ph.D, mine.D, ph.dtype, mine.dtype, ph.world, mine.world);
        c->peer_remote[j] = std::memcmp(ph.uuid, mine.uuid, sizeof(mine.uuid)) != 0;
        c->peers[j].k = b;
        c->peers[j].v = b + c->off_v;
        c->peers[j].pos = reinterpret_cast<int32_t*>(b + c->off_pos);
        c->peers[j].flags = reinterpret_cast<unsigned long long*>(b + c->off_flags);
    }
    c->connected = true;
    return CDSP_OK;
}

cdsp_status cdsp_comm_connect_local(cdsp_comm* comms, int32_t world) {
    CDSP_REQUIRE(comms != nullptr && world >= 1 && world <= kMaxWorld, CDSP_ERR_INVALID, "bad comms/world");
    for (int i = 0; i < world; ++i) {
        CDSP_REQUIRE(comms[i] != nullptr, CDSP_ERR_INVALID, "comms[%d] is NULL", i);
        CDSP_REQUIRE(comms[i]->rank == i && comms[i]->world == world, CDSP_ERR_INVALID,
                     "comms[%d] has rank %d / world %d", i, comms[i]->rank, comms[i]->world);
        CDSP_REQUIRE(comms[i]->cap == comms[0]->cap && comms[i]->n_layers == comms[0]->n_layers &&
                         comms[i]->Hkv == comms[0]->Hkv &&
                         comms[i]->D == comms[0]->D && comms[i]->dtype == comms[0]->dtype &&
                         comms[i]->device == comms[0]->device,
                     CDSP_ERR_INVALID, "loopback communicators must share geometry and device");
        CDSP_REQUIRE(!comms[i]->connected && comms[i]->lg == nullptr, CDSP_ERR_INVALID,
                     "comms[%d] is already connected", i);
    }
    LocalGroup* g = new LocalGroup();
    g->world = world;
    g->refs = world;
    for (int i = 0; i < world; ++i) {
        g->comms[i] = comms[i];
        for (int j = 0; j < world; ++j) comms[i]->peers[j] = comms[j]->self;
        comms[i]->connected = true;
        comms[i]->lg = g;
    }
    return CDSP_OK;
}

cdsp_status cdsp_comm_check(cdsp_comm c) {
    CDSP_REQUIRE(c != nullptr, CDSP_ERR_INVALID, "NULL comm");
    if (*reinterpret_cast<volatile int*>(c->err_host) != 0)
        CDSP_FAIL(CDSP_ERR_COMM, "peer barrier timed out on instance %d", c->rank);
    return CDSP_OK;
}

cdsp_status cdsp_comm_profile(cdsp_comm c, int32_t enable) {
    CDSP_REQUIRE(c != nullptr, CDSP_ERR_INVALID, "NULL comm");
    if (enable && c->prof_ev.empty()) {
        c->prof_ev.resize(2 * 8192, nullptr);
        for (auto& ev : c->prof_ev) CDSP_CUDA(cudaEventCreate(&ev));
        c->ring_ev.resize(2 * 4096, nullptr);
        for (auto& ev : c->ring_ev) CDSP_CUDA(cudaEventCreate(&ev));
        c->ring_rec.resize(4096);
        CDSP_CUDA(cudaEventCreate(&c->ev_ring0));
    }
    c->profiling = enable != 0;
    c->prof_n = 0;
    c->ring_n = 0;
    return CDSP_OK;
}

cdsp_status cdsp_comm_profile_ring(cdsp_comm c, double* copy_ms, double* exposed_ms, int64_t* bytes,
                                   int32_t* n_pulls) {
    CDSP_REQUIRE(c && copy_ms && exposed_ms && bytes && n_pulls, CDSP_ERR_INVALID, "NULL argument");
    double cp = 0.0, ex = 0.0;
    int64_t by = 0;
    if (c->ring_n > 0) CDSP_CUDA(cudaEventSynchronize(c->ring_ev[2 * c->ring_n - 1]));
    for (int i = 0; i < c->ring_n; ++i) {
        const auto& r = c->ring_rec[i];
        float ms = 0.f;
        CDSP_CUDA(cudaEventElapsedTime(&ms, c->ring_ev[2 * r.ev], c->ring_ev[2 * r.ev + 1]));
        cp += ms;
        by += r.bytes;
        if (r.from != nullptr) {
            // the compute stream idles from `from` (the previous launch's end, or the ring's
            // start) until this pull lands: its next launch waits on it
            CDSP_CUDA(cudaEventSynchronize(r.from));
            float gap = 0.f;
            CDSP_CUDA(cudaEventElapsedTime(&gap, r.from, c->ring_ev[2 * r.ev + 1]));
            if (gap > 0.f) ex += gap;
        }
    }
    *copy_ms = cp;
    *exposed_ms = ex;
    *bytes = by;
    *n_pulls = c->ring_n;
    c->ring_n = 0;
    return CDSP_OK;
}

cdsp_status cdsp_comm_profile_read(cdsp_comm c, double* attn_ms, int32_t* n_launches) {
    CDSP_REQUIRE(c && attn_ms && n_launches, CDSP_ERR_INVALID, "NULL argument");
    double total = 0.0;
    if (c->prof_n > 0) CDSP_CUDA(cudaEventSynchronize(c->prof_ev[2 * c->prof_n - 1]));
    for (int i = 0; i < c->prof_n; ++i) {
        float ms = 0.f;
        CDSP_CUDA(cudaEventElapsedTime(&ms, c->prof_ev[2 * i], c->prof_ev[2 * i + 1]));
        total += ms;
    }
    *attn_ms = total;
    *n_launches = c->prof_n;
    c->prof_n = 0;
    return CDSP_OK;
}

cdsp_status cdsp_comm_destroy(cdsp_comm c) {
    if (!c) return CDSP_OK;
    cudaDeviceSynchronize();
    for (auto ev : c->prof_ev)
        if (ev) cudaEventDestroy(ev);
    for (auto ev : c->ring_ev)
        if (ev) cudaEventDestroy(ev);
    for (auto ev : c->ev_bal_l)
        if (ev) cudaEventDestroy(ev);
    for (int j = 0; j < kMaxWorld; ++j)
        if (c->ipc_base[j]) cudaIpcCloseMemHandle(c->ipc_base[j]);
    if (c->o_acc) cudaFree(c->o_acc);
    if (c->lse_acc) cudaFree(c->lse_acc);
    if (c->recv) cudaFree(c->recv);
    if (c->gate) cudaFree(c->gate);
    if (c->ev_ring0) cudaEventDestroy(c->ev_ring0);
    for (auto ev : c->ev_pull)
        if (ev) cudaEventDestroy(ev);
    if (c->region) cudaFree(c->region);
    if (c->bad_count) cudaFree(c->bad_count);
    if (c->err_host) cudaFreeHost(c->err_host);
    if (c->lg && --c->lg->refs == 0) delete c->lg;
    cudaEvent_t evs[7] = {c->ev_ready, c->ev_done, c->ev_bal, c->ev_app, c->ev_fin, c->ev_x0, c->ev_x1};
    for (auto ev : evs)
        if (ev) cudaEventDestroy(ev);
    if (c->comm_stream) cudaStreamDestroy(c->comm_stream);
    if (c->xfer_stream) cudaStreamDestroy(c->xfer_stream);
    delete c;
    return CDSP_OK;
}

cdsp_status cdsp_kvstore_get(cdsp_comm c, cdsp_kvstore* out) { return cdsp_kvstore_get_layer(c, 0, out); }

cdsp_status cdsp_kvstore_get_layer(cdsp_comm c, int32_t layer, cdsp_kvstore* out) {
    CDSP_REQUIRE(c && out, CDSP_ERR_INVALID, "NULL argument");
    CDSP_REQUIRE(layer >= 0 && layer < c->n_layers, CDSP_ERR_INVALID, "layer %d not in [0,%d)", layer, c->n_layers);
    out->k = cdsp_tensor{layer_k(c, c->self, layer), c->dtype, c->cap, c->Hkv, c->D};
    out->v = cdsp_tensor{layer_v(c, c->self, layer), c->dtype, c->cap, c->Hkv, c->D};
    out->pos = c->self.pos;
    out->n = c->n_l[layer];
    out->cap = c->cap;
    return CDSP_OK;
}

cdsp_status cdsp_kvstore_reset(cdsp_comm c, void* cuda_stream) {
    CDSP_REQUIRE(c != nullptr, CDSP_ERR_INVALID, "NULL comm");
    (void)cuda_stream;  // content is overwritten in stream order by the next chunk
    for (auto& n : c->n_l) n = 0;
    for (auto& pb : c->prebal) pb = -1;
    c->prebal_plan = nullptr;
    return CDSP_OK;
}

// ------------------------------------------------------------------------------- plan
cdsp_status cdsp_plan_capacity(const cdsp_plan* plan, int64_t* rows) {
    CDSP_REQUIRE(rows != nullptr, CDSP_ERR_INVALID, "rows is NULL");
    ChunkInfo ci;
    CDSP_CHECK_STATUS(plan_chunk_info(plan, 0, &ci));  // validates the plan
    *rows = plan_max_store(plan);
    return CDSP_OK;
}

cdsp_status cdsp_plan_partition(const cdsp_plan* plan, int32_t c, int32_t* tok_rank, int32_t* tok_slot,
                                int64_t* rank_pos, cdsp_move* moves, int32_t* n_moves) {
    ChunkInfo ci;
    CDSP_CHECK_STATUS(plan_chunk_info(plan, c, &ci));
    const int64_t m = ci.m;
    const bool striped = ci.interleave == CDSP_STRIPED;
    if (tok_rank || tok_slot) {
        for (int64_t t = 0; t < ci.L; ++t) {
            if (striped) {  // round-robin stripes (R20)
                if (tok_rank) tok_rank[t] = static_cast<int32_t>(t % ci.s);
                if (tok_slot) tok_slot[t] = static_cast<int32_t>(t / ci.s);
                continue;
            }
            const int64_t j = t / m;  // shard S_j
            const bool first = j < ci.s;
            if (tok_rank) tok_rank[t] = static_cast<int32_t>(first ? j : 2 * ci.s - 1 - j);
            if (tok_slot) tok_slot[t] = static_cast<int32_t>(first ? t - j * m : m + (t - j * m));
        }
    }
    if (rank_pos) {
        const int64_t st = shard_stride(ci);
        for (int r = 0; r < ci.s; ++r) {
            int64_t* p = rank_pos + static_cast<size_t>(r) * 2 * m;
            for (int64_t i = 0; i < m; ++i) {
                p[i] = shard_pos0(ci, r) + i * st;
                p[m + i] = shard_pos1(ci, r) + i * st;
            }
        }
    }
    if (moves)
        for (int i = 0; i < ci.n_moves; ++i) moves[i] = ci.moves[i];
    if (n_moves) *n_moves = ci.n_moves;
    return CDSP_OK;
}

// ------------------------------------------------------------------------------- prefill
cdsp_status cdsp_prefill_chunk(const cdsp_tensor* q, const cdsp_tensor* k, const cdsp_tensor* v,
                               cdsp_kvstore* prev_kv, const cdsp_sp_group* sp_group, float softmax_scale,
                               cdsp_tensor* out, float* lse, void* cuda_stream) {
    return cdsp_prefill_chunk_layer(q, k, v, prev_kv, sp_group, 0, softmax_scale, out, lse, cuda_stream);
}

namespace cdsp {
namespace {
// The decode target's checks shared by cdsp_kv_transfer_to_decode and the fused path.
static cdsp_status check_decode_target(const cdsp_decode_target* dst, const cdsp_tensor* k, const ChunkInfo& ci) {
    CDSP_REQUIRE(dst->tp >= 1 && dst->tp <= 8, CDSP_ERR_INVALID, "decode tp %d not in [1,8]", dst->tp);
    CDSP_REQUIRE(k->H % dst->tp == 0, CDSP_ERR_UNSUPPORTED,
                 "Hkv=%lld not divisible by decode tp=%d (KV-head replication is not defined)",
                 static_cast<long long>(k->H), dst->tp);
    CDSP_REQUIRE(dst->block_size >= 1 && dst->num_blocks >= 1 && dst->block_table && dst->k_cache && dst->v_cache,
                 CDSP_ERR_INVALID, "bad decode target");
    CDSP_REQUIRE(dst->n_table * dst->block_size >= ci.C + ci.L, CDSP_ERR_CAPACITY,
                 "block table covers %lld positions, chunk ends at %lld",
                 static_cast<long long>(dst->n_table * dst->block_size), static_cast<long long>(ci.C + ci.L));
    for (int t = 0; t < dst->tp; ++t)
        CDSP_REQUIRE(dst->k_cache[t] && dst->v_cache[t], CDSP_ERR_INVALID, "NULL cache pointer for tp rank %d", t);
    return CDSP_OK;
}

static cdsp_status prefill_impl(const cdsp_tensor* q, const cdsp_tensor* k, const cdsp_tensor* v, cdsp_kvstore* prev_kv,
                                const cdsp_sp_group* sp_group, int32_t layer, float softmax_scale, cdsp_tensor* out,
                                float* lse, void* cuda_stream);
}  // namespace
}  // namespace cdsp

cdsp_status cdsp_prefill_chunk_layer(const cdsp_tensor* q, const cdsp_tensor* k, const cdsp_tensor* v,
                                     cdsp_kvstore* prev_kv, const cdsp_sp_group* sp_group, int32_t layer,
                                     float softmax_scale, cdsp_tensor* out, float* lse, void* cuda_stream) {
    return prefill_impl(q, k, v, prev_kv, sp_group, layer, softmax_scale, out, lse, cuda_stream);
}

cdsp_status cdsp_prefill_chunk_transfer(const cdsp_tensor* q, const cdsp_tensor* k, const cdsp_tensor* v,
                                        cdsp_kvstore* prev_kv, const cdsp_sp_group* sp_group, float softmax_scale,
                                        cdsp_tensor* out, float* lse, const cdsp_decode_target* dst,
                                        void* cuda_stream) {
    CDSP_REQUIRE(dst != nullptr && sp_group && sp_group->comm && sp_group->plan, CDSP_ERR_INVALID,
                 "NULL decode target / group");
    cdsp_comm c = sp_group->comm;
    {  // the transfer's own checks first: a refused call enqueues nothing
        CDSP_CHECK_STATUS(check_tensor(k, "k"));
        ChunkInfo ci;
        CDSP_CHECK_STATUS(plan_chunk_info(sp_group->plan, sp_group->chunk, &ci));
        CDSP_CHECK_STATUS(check_decode_target(dst, k, ci));
    }
    cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
    CDSP_CUDA(cudaEventRecord(c->ev_x0, st));  // this call's k / v are ready
    // the attention first: its persistent grid takes every SM; the scatter, on the comm's
    // transfer stream, fills SMs as the attention's tail frees them (enqueued first, its CTAs
    // would hold SMs the attention needs)
    CDSP_CHECK_STATUS(prefill_impl(q, k, v, prev_kv, sp_group, 0, softmax_scale, out, lse, cuda_stream));
    // measurement control CDSP_XFER_SERIAL=1: the scatter after the attention on the caller's stream
    static const bool serial = getenv("CDSP_XFER_SERIAL") != nullptr && getenv("CDSP_XFER_SERIAL")[0] == '1';
    if (serial) return cdsp_kv_transfer_to_decode(k, v, sp_group, dst, cuda_stream);
    CDSP_CUDA(cudaStreamWaitEvent(c->xfer_stream, c->ev_x0, 0));
    CDSP_CHECK_STATUS(cdsp_kv_transfer_to_decode(k, v, sp_group, dst, c->xfer_stream));
    CDSP_CUDA(cudaEventRecord(c->ev_x1, c->xfer_stream));
    CDSP_CUDA(cudaStreamWaitEvent(st, c->ev_x1, 0));  // the caller's stream sees both
    return CDSP_OK;
}

namespace cdsp {
namespace {
static cdsp_status prefill_impl(const cdsp_tensor* q, const cdsp_tensor* k, const cdsp_tensor* v, cdsp_kvstore* prev_kv,
                                const cdsp_sp_group* sp_group, int32_t layer, float softmax_scale, cdsp_tensor* out,
                                float* lse, void* cuda_stream) {
    CDSP_REQUIRE(sp_group && sp_group->comm && sp_group->plan && prev_kv, CDSP_ERR_INVALID,
                 "NULL sp_group/comm/plan/prev_kv");
    CDSP_CHECK_STATUS(check_tensor(q, "q"));
    CDSP_CHECK_STATUS(check_tensor(k, "k"));
    CDSP_CHECK_STATUS(check_tensor(v, "v"));
    CDSP_CHECK_STATUS(check_tensor(out, "out"));
    cdsp_comm c = sp_group->comm;
    ChunkInfo ci;
    CDSP_CHECK_STATUS(plan_chunk_info(sp_group->plan, sp_group->chunk, &ci));
    const int r = plan_ring_rank(ci, c->rank);
    CDSP_REQUIRE(r >= 0, CDSP_ERR_PLAN, "instance %d is not in chunk %d's group", c->rank, ci.c);
    for (int i = 0; i < ci.s; ++i)
        CDSP_REQUIRE(ci.ranks[i] < c->world, CDSP_ERR_PLAN, "plan names instance %d >= world %d", ci.ranks[i],
                     c->world);
    const int64_t m2 = 2 * ci.m;
    CDSP_REQUIRE(q->dtype == k->dtype && k->dtype == v->dtype && out->dtype == q->dtype && q->dtype == c->dtype,
                 CDSP_ERR_DTYPE, "q/k/v/out/store dtypes differ");
    CDSP_REQUIRE(q->T == m2 && k->T == m2 && v->T == m2 && out->T == m2, CDSP_ERR_SHAPE,
                 "q/k/v/out must hold the rank's 2m=%lld shard rows", static_cast<long long>(m2));
    CDSP_REQUIRE(q->D == c->D && k->D == c->D && v->D == c->D && out->D == c->D, CDSP_ERR_SHAPE,
                 "head dim mismatch");
    CDSP_REQUIRE(k->H == c->Hkv && v->H == c->Hkv, CDSP_ERR_SHAPE, "k/v heads must equal store Hkv=%d", c->Hkv);
    CDSP_REQUIRE(q->H % c->Hkv == 0 && out->H == q->H, CDSP_ERR_SHAPE, "Hq %% Hkv != 0 or out heads != Hq");
    CDSP_REQUIRE(layer >= 0 && layer < c->n_layers, CDSP_ERR_INVALID, "layer %d not in [0,%d)", layer, c->n_layers);
    CDSP_REQUIRE(prev_kv->k.ptr == layer_k(c, c->self, layer) && prev_kv->v.ptr == layer_v(c, c->self, layer),
                 CDSP_ERR_INVALID, "prev_kv is not this communicator's layer-%d store (use cdsp_kvstore_get_layer)",
                 layer);
    CDSP_REQUIRE(c->n_l[layer] == ci.store_before[r], CDSP_ERR_PLAN,
                 "layer %d store holds %lld rows but the plan expects %lld before chunk %d (missing "
                 "cdsp_kvstore_reset?)",
                 layer, static_cast<long long>(c->n_l[layer]), static_cast<long long>(ci.store_before[r]), ci.c);
    for (int i = 0; i < ci.s; ++i)
        CDSP_REQUIRE(ci.hist[i] + m2 <= c->cap, CDSP_ERR_CAPACITY,
                     "ring rank %d needs %lld store rows, capacity %lld", i,
                     static_cast<long long>(ci.hist[i] + m2), static_cast<long long>(c->cap));
    CDSP_REQUIRE(ci.s == 1 || c->connected, CDSP_ERR_INVALID, "communicator not connected");
    CDSP_CHECK_STATUS(cdsp_comm_check(c));
    cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
    const float scale = softmax_scale > 0.f ? softmax_scale : 1.0f / sqrtf(static_cast<float>(c->D));
    const int Hq = static_cast<int>(q->H);
    if (ci.s > 1) {  // the ring's launch structure; several launches merge through the reserved accumulators
        RingLaunches rl;
        CDSP_CHECK_STATUS(ring_launches(c, ci, r, &rl, Hq));
        CDSP_REQUIRE(rl.n == 1 || (c->acc_rows >= m2 && c->acc_hq >= Hq), CDSP_ERR_CAPACITY,
                     "this ring runs as %d launches merged in fp32 accumulators: reserve %lld rows x %d heads with "
                     "cdsp_comm_reserve (reserved %lld x %d)",
                     rl.n, static_cast<long long>(m2), Hq, static_cast<long long>(c->acc_rows), c->acc_hq);
        CDSP_REQUIRE(ci.s - 1 <= c->n_slots, CDSP_ERR_INVALID, "ring of %d needs %d receive slots, comm has %d", ci.s,
                     ci.s - 1, c->n_slots);
    }

    if (ci.s > 1 && c->lg != nullptr) {
        // loopback: a deferred collective (like an NCCL group) — record this rank's call; the
        // call that completes the group issues every rank's phases in dependency order, with
        // CUDA events instead of device-side peer barriers
        LocalGroup* g = c->lg;
        CDSP_REQUIRE(g->pending == 0 ||
                         (g->plan == sp_group->plan && g->chunk == sp_group->chunk && g->layer == layer),
                     CDSP_ERR_INVALID, "loopback group has a pending call for another chunk / layer");
        CDSP_REQUIRE(!g->calls[r].set, CDSP_ERR_INVALID, "ring rank %d already called chunk %d", r, ci.c);
        g->plan = sp_group->plan;
        g->chunk = sp_group->chunk;
        g->layer = layer;
        g->calls[r] = PendingCall{layer, *q, *k, *v, *out, lse, prev_kv, scale, st, true};
        if (++g->pending < ci.s) return CDSP_OK;
        g->pending = 0;
        cdsp_status rc = run_group_local(g, ci, layer);
        for (int i = 0; i < ci.s; ++i) g->calls[i].set = false;
        return rc;
    }

    // B1 (once per chunk: every peer finished the previous chunk, all layers)
    if (ci.s > 1 && layer == 0) CDSP_CHECK_STATUS(barrier(c, ci, st));
    // cache balancing (R8) of this layer, unless the previous layer pre-issued it
    if (balancing(ci)) {
        if (prebalanced(c, ci, layer, sp_group->plan))
            CDSP_CUDA(cudaStreamWaitEvent(st, c->ev_bal_l[layer], 0));
        else
            CDSP_CHECK_STATUS(phase_balance_pull(c, ci, r, layer, st, true));
        CDSP_CHECK_STATUS(phase_balance_wait(c, ci, r, st));  // sources: pullers are done with it
    }
    int64_t& n = c->n_l[layer];
    n = ci.hist[r];
    if (ci.s == 1 && n == 0) {
        // single instance, no history: the attention reads this call's k/v directly while the
        // copy engines append them to the store on the comm stream (no SMs taken from it)
        CDSP_CUDA(cudaEventRecord(c->ev_ready, st));
        CDSP_CUDA(cudaStreamWaitEvent(c->comm_stream, c->ev_ready, 0));
        CDSP_CUDA(cudaMemcpyAsync(layer_k(c, c->self, layer), k->ptr, m2 * c->row_bytes, cudaMemcpyDeviceToDevice,
                                  c->comm_stream));
        CDSP_CUDA(cudaMemcpyAsync(layer_v(c, c->self, layer), v->ptr, m2 * c->row_bytes, cudaMemcpyDeviceToDevice,
                                  c->comm_stream));
        CDSP_CHECK_STATUS(launch_fill_positions(c->self.pos, m2, ci.m, shard_pos0(ci, r), shard_pos1(ci, r),
                                                shard_stride(ci), c->comm_stream));
        n = m2;
        prev_kv->n = n;
        AttnArgs a = attn_args(c, q->ptr, Hq, scale, CDSP_ATTN_ONLY, out->ptr, lse);
        a.k[0] = k->ptr;
        a.v[0] = v->ptr;
        a.seg[0] = segments_for(ci, r, 0);
        CDSP_CHECK_STATUS(run_attention_timed(c, a, st));
        CDSP_CUDA(cudaEventRecord(c->ev_done, c->comm_stream));
        CDSP_CUDA(cudaStreamWaitEvent(st, c->ev_done, 0));
        return CDSP_OK;
    }
    CDSP_CHECK_STATUS(phase_append(c, ci, r, layer, k, v, st));
    prev_kv->n = n;
    if (ci.s == 1) {
        AttnArgs a = attn_args(c, q->ptr, Hq, scale, CDSP_ATTN_ONLY, out->ptr, lse);
        a.k[0] = layer_k(c, c->self, layer);
        a.v[0] = layer_v(c, c->self, layer);
        a.seg[0] = segments_for(ci, r, 0);
        return run_attention_timed(c, a, st);
    }
    CDSP_CHECK_STATUS(barrier(c, ci, st));  // B3
    CDSP_CHECK_STATUS(phase_ring(c, ci, r, layer, q->ptr, Hq, out->ptr, lse, scale, st, nullptr));
    return prebalance_next(c, ci, r, layer, sp_group->plan, true);
}
}  // namespace
}  // namespace cdsp

// ------------------------------------------------------------------------------- merge
cdsp_status cdsp_lse_merge(int32_t n, const cdsp_tensor* const* o_parts, const float* const* lse_parts,
                           cdsp_tensor* out, float* lse, void* cuda_stream) {
    CDSP_REQUIRE(n >= 1 && n <= kMaxMerge, CDSP_ERR_INVALID, "n=%d not in [1,%d]", n, kMaxMerge);
    CDSP_REQUIRE(o_parts && lse_parts, CDSP_ERR_INVALID, "NULL parts");
    CDSP_CHECK_STATUS(check_tensor(out, "out"));
    const float* ptrs[kMaxMerge];
    for (int i = 0; i < n; ++i) {
        CDSP_CHECK_STATUS(check_tensor(o_parts[i], "o_parts[i]"));
        CDSP_REQUIRE(o_parts[i]->dtype == CDSP_F32, CDSP_ERR_DTYPE, "partials must be fp32");
        CDSP_REQUIRE(o_parts[i]->T == out->T && o_parts[i]->H == out->H && o_parts[i]->D == out->D, CDSP_ERR_SHAPE,
                     "part %d shape differs from out", i);
        CDSP_REQUIRE(lse_parts[i] != nullptr || out->T == 0, CDSP_ERR_INVALID, "lse_parts[%d] is NULL", i);
        ptrs[i] = static_cast<const float*>(o_parts[i]->ptr);
    }
    CDSP_REQUIRE(out->D == 64 || out->D == 128, CDSP_ERR_SHAPE, "head dim %lld not in {64,128}",
                 static_cast<long long>(out->D));
    return launch_lse_merge(n, ptrs, lse_parts, out->T, static_cast<int>(out->H), static_cast<int>(out->D),
                            out->ptr, out->dtype, lse, static_cast<cudaStream_t>(cuda_stream));
}

// ------------------------------------------------------------------------------- KV transfer
cdsp_status cdsp_kv_transfer_to_decode(const cdsp_tensor* k, const cdsp_tensor* v, const cdsp_sp_group* sp_group,
                                       const cdsp_decode_target* dst, void* cuda_stream) {
    CDSP_REQUIRE(sp_group && sp_group->comm && sp_group->plan && dst, CDSP_ERR_INVALID, "NULL argument");
    CDSP_CHECK_STATUS(check_tensor(k, "k"));
    CDSP_CHECK_STATUS(check_tensor(v, "v"));
    cdsp_comm c = sp_group->comm;
    ChunkInfo ci;
    CDSP_CHECK_STATUS(plan_chunk_info(sp_group->plan, sp_group->chunk, &ci));
    const int r = plan_ring_rank(ci, c->rank);
    CDSP_REQUIRE(r >= 0, CDSP_ERR_PLAN, "instance %d is not in chunk %d's group", c->rank, ci.c);
    CDSP_REQUIRE(k->dtype == v->dtype, CDSP_ERR_DTYPE, "k/v dtypes differ");
    CDSP_REQUIRE(k->T == 2 * ci.m && v->T == k->T && v->H == k->H && v->D == k->D, CDSP_ERR_SHAPE,
                 "k/v must be this rank's [2m, Hkv, D] shard");
    CDSP_CHECK_STATUS(check_decode_target(dst, k, ci));
    PagedArgs a;
    std::memset(&a, 0, sizeof(a));
    a.k = k->ptr;
    a.v = v->ptr;
    a.n_tok = k->T;
    a.Hkv = static_cast<int>(k->H);
    a.D = static_cast<int>(k->D);
    a.esize = static_cast<int>(dtype_size(k->dtype));
    a.len0 = ci.m;
    a.pos0 = shard_pos0(ci, r);
    a.pos1 = shard_pos1(ci, r);
    a.pos_stride = shard_stride(ci);
    a.tp = dst->tp;
    a.block_size = dst->block_size;
    a.num_blocks = dst->num_blocks;
    a.n_table = dst->n_table;
    a.block_table = dst->block_table;
    for (int t = 0; t < dst->tp; ++t) {
        a.k_cache[t] = dst->k_cache[t];
        a.v_cache[t] = dst->v_cache[t];
    }
    a.bad_count = c->bad_count;
    cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
    CDSP_CUDA(cudaMemsetAsync(c->bad_count, 0, sizeof(unsigned long long), st));
    return launch_paged_scatter(a, st);
}

cdsp_status cdsp_kv_transfer_errors(cdsp_comm c, void* cuda_stream, int64_t* n_bad) {
    CDSP_REQUIRE(c && n_bad, CDSP_ERR_INVALID, "NULL argument");
    unsigned long long h = 0;
    cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
    CDSP_CUDA(cudaMemcpyAsync(&h, c->bad_count, sizeof(h), cudaMemcpyDeviceToHost, st));
    CDSP_CUDA(cudaStreamSynchronize(st));
    *n_bad = static_cast<int64_t>(h);
    return CDSP_OK;
}

// ------------------------------------------------------------------------------- blocks
cdsp_status cdsp_attention_fwd_blocks(const cdsp_tensor* q, int32_t nblk, const cdsp_tensor* const* k,
                                      const cdsp_tensor* const* v, const cdsp_segments* seg, float softmax_scale,
                                      int32_t mode, float* o_acc, float* lse_acc, cdsp_tensor* out, float* lse,
                                      void* cuda_stream) {
    CDSP_REQUIRE(nblk >= 1 && nblk <= CDSP_MAX_SP, CDSP_ERR_INVALID, "nblk %d not in [1,%d]", nblk, CDSP_MAX_SP);
    CDSP_REQUIRE(k != nullptr && v != nullptr && seg != nullptr, CDSP_ERR_INVALID, "NULL k/v/segments");
    const bool pdl = (mode & CDSP_ATTN_PDL) != 0;
    mode &= ~CDSP_ATTN_PDL;
    CDSP_REQUIRE(mode >= CDSP_ATTN_ONLY && mode <= CDSP_ATTN_LAST, CDSP_ERR_INVALID, "bad mode %d", mode);
    CDSP_CHECK_STATUS(check_tensor(q, "q"));
    CDSP_REQUIRE(q->D == 64 || q->D == 128, CDSP_ERR_SHAPE, "head dim must be 64 or 128");
    CDSP_REQUIRE(q->dtype == CDSP_BF16 || nblk == 1, CDSP_ERR_UNSUPPORTED, "fp32 attention takes one KV block per launch");
    AttnArgs a;
    a.nblk = nblk;
    int64_t tiles = 0;
    for (int b = 0; b < nblk; ++b) {
        CDSP_REQUIRE(k[b] != nullptr && v[b] != nullptr, CDSP_ERR_INVALID, "NULL k/v of block %d", b);
        CDSP_CHECK_STATUS(check_tensor(k[b], "k"));
        CDSP_CHECK_STATUS(check_tensor(v[b], "v"));
        const cdsp_segments& sb = seg[b];
        CDSP_REQUIRE(sb.pos_stride >= 0 && sb.pos_stride <= 8, CDSP_ERR_SHAPE, "pos_stride %lld not in [0,8]",
                     static_cast<long long>(sb.pos_stride));
        CDSP_REQUIRE(q->dtype == k[b]->dtype && k[b]->dtype == v[b]->dtype, CDSP_ERR_DTYPE, "q/k/v dtypes differ");
        CDSP_REQUIRE(q->D == k[b]->D && k[b]->D == v[b]->D, CDSP_ERR_SHAPE, "head dims differ");
        CDSP_REQUIRE(k[b]->H == v[b]->H && k[b]->H == k[0]->H && q->H % k[b]->H == 0, CDSP_ERR_SHAPE,
                     "Hq %% Hkv != 0 or KV heads differ between blocks");
        CDSP_REQUIRE(sb.nq == q->T && sb.nkv <= k[b]->T && sb.nkv <= v[b]->T && sb.nkv >= 0, CDSP_ERR_SHAPE,
                     "segments of block %d do not match tensor rows", b);
        CDSP_REQUIRE(sb.q_len0 >= 0 && sb.q_len0 <= sb.nq && sb.kv_hist >= 0 && sb.kv_len0 >= 0 &&
                         sb.kv_hist + sb.kv_len0 <= sb.nkv,
                     CDSP_ERR_SHAPE, "inconsistent segments (block %d)", b);
        CDSP_REQUIRE(sb.q_len0 == seg[0].q_len0 && sb.q_pos0 == seg[0].q_pos0 && sb.q_pos1 == seg[0].q_pos1 &&
                         (sb.pos_stride ? sb.pos_stride : 1) == (seg[0].pos_stride ? seg[0].pos_stride : 1),
                     CDSP_ERR_SHAPE, "block %d's query segments differ from block 0's", b);
        a.k[b] = k[b]->ptr;
        a.v[b] = v[b]->ptr;
        a.seg[b] = sb;
        if (a.seg[b].pos_stride == 0) a.seg[b].pos_stride = 1;  // 0 = contiguous (ABI 1 callers)
        tiles += (sb.nkv + 127) / 128;
    }
    if (q->dtype == CDSP_BF16)
        CDSP_REQUIRE(tiles <= attention_tc_max_tiles(static_cast<int>(q->D)), CDSP_ERR_CAPACITY,
                     "%lld KV tiles exceed the %d of one launch (split the blocks with FIRST / MID / LAST)",
                     static_cast<long long>(tiles), attention_tc_max_tiles(static_cast<int>(q->D)));
    const bool final_out = mode == CDSP_ATTN_ONLY || mode == CDSP_ATTN_LAST;
    if (final_out) {
        CDSP_CHECK_STATUS(check_tensor(out, "out"));
        CDSP_REQUIRE(out->dtype == q->dtype && out->T == q->T && out->H == q->H && out->D == q->D, CDSP_ERR_SHAPE,
                     "out must match q");
    }
    CDSP_REQUIRE(mode == CDSP_ATTN_ONLY || (o_acc && lse_acc) || q->T == 0, CDSP_ERR_INVALID,
                 "accumulator buffers required for mode %d", mode);
    a.q = q->ptr;
    a.dtype = q->dtype;
    a.Hq = static_cast<int>(q->H);
    a.Hkv = static_cast<int>(k[0]->H);
    a.D = static_cast<int>(q->D);
    a.scale = softmax_scale > 0.f ? softmax_scale : 1.0f / sqrtf(static_cast<float>(q->D));
    a.mode = mode;
    a.o_acc = o_acc;
    a.lse_acc = lse_acc;
    a.out = final_out ? out->ptr : nullptr;
    a.lse = lse;
    a.pdl = pdl;
    a.split_ok = mode == CDSP_ATTN_ONLY && o_acc && lse_acc;  // scratch given: heavy units may split
    return run_attention(a, static_cast<cudaStream_t>(cuda_stream));
}

cdsp_status cdsp_attention_fwd(const cdsp_tensor* q, const cdsp_tensor* k, const cdsp_tensor* v,
                               const cdsp_segments* seg, float softmax_scale, int32_t mode, float* o_acc,
                               float* lse_acc, cdsp_tensor* out, float* lse, void* cuda_stream) {
    return cdsp_attention_fwd_blocks(q, 1, &k, &v, seg, softmax_scale, mode, o_acc, lse_acc, out, lse, cuda_stream);
}

static cdsp_status zigzag_copy(const cdsp_tensor* full, int32_t s, int32_t r, cdsp_tensor* shard, bool gather,
                               cudaStream_t st) {
    CDSP_CHECK_STATUS(check_tensor(full, "full"));
    CDSP_CHECK_STATUS(check_tensor(shard, "shard"));
    CDSP_REQUIRE(s == 1 || s == 2 || s == 4 || s == 8, CDSP_ERR_PLAN, "s=%d not in {1,2,4,8}", s);
    CDSP_REQUIRE(r >= 0 && r < s, CDSP_ERR_INVALID, "rank %d not in [0,%d)", r, s);
    CDSP_REQUIRE(full->dtype == shard->dtype, CDSP_ERR_DTYPE, "dtype mismatch");
    CDSP_REQUIRE(full->H == shard->H && full->D == shard->D, CDSP_ERR_SHAPE, "H/D mismatch");
    CDSP_REQUIRE(full->T % (2 * s) == 0, CDSP_ERR_SHAPE, "L=%lld not a multiple of 2s", static_cast<long long>(full->T));
    const int64_t m = full->T / (2 * s);
    CDSP_REQUIRE(shard->T == 2 * m, CDSP_ERR_SHAPE, "shard must have 2m=%lld rows", static_cast<long long>(2 * m));
    const int64_t row_bytes = full->H * full->D * static_cast<int64_t>(dtype_size(full->dtype));
    RowCopy segs[2];
    const int64_t f0 = static_cast<int64_t>(r) * m, f1 = static_cast<int64_t>(2 * s - 1 - r) * m;
    if (gather) {
        segs[0] = RowCopy{full->ptr, shard->ptr, f0, 0, m};
        segs[1] = RowCopy{full->ptr, shard->ptr, f1, m, m};
    } else {
        segs[0] = RowCopy{shard->ptr, full->ptr, 0, f0, m};
        segs[1] = RowCopy{shard->ptr, full->ptr, m, f1, m};
    }
    return launch_row_copy(segs, 2, row_bytes, st);
}

static cdsp_status striped_copy(const cdsp_tensor* full, int32_t s, int32_t r, cdsp_tensor* shard, bool gather,
                                cudaStream_t st) {
    CDSP_CHECK_STATUS(check_tensor(full, "full"));
    CDSP_CHECK_STATUS(check_tensor(shard, "shard"));
    CDSP_REQUIRE(s == 1 || s == 2 || s == 4 || s == 8, CDSP_ERR_PLAN, "s=%d not in {1,2,4,8}", s);
    CDSP_REQUIRE(r >= 0 && r < s, CDSP_ERR_INVALID, "rank %d not in [0,%d)", r, s);
    CDSP_REQUIRE(full->dtype == shard->dtype, CDSP_ERR_DTYPE, "dtype mismatch");
    CDSP_REQUIRE(full->H == shard->H && full->D == shard->D, CDSP_ERR_SHAPE, "H/D mismatch");
    CDSP_REQUIRE(full->T % (2 * s) == 0, CDSP_ERR_SHAPE, "L=%lld not a multiple of 2s", static_cast<long long>(full->T));
    const int64_t n = full->T / s;
    CDSP_REQUIRE(shard->T == n, CDSP_ERR_SHAPE, "shard must have L/s=%lld rows", static_cast<long long>(n));
    const int64_t row_bytes = full->H * full->D * static_cast<int64_t>(dtype_size(full->dtype));
    RowCopy seg = gather ? RowCopy{full->ptr, shard->ptr, r, 0, n, s, 1} : RowCopy{shard->ptr, full->ptr, 0, r, n, 1, s};
    return launch_row_copy(&seg, 1, row_bytes, st);
}

cdsp_status cdsp_striped_gather(const cdsp_tensor* full, int32_t s, int32_t r, cdsp_tensor* shard, void* cuda_stream) {
    return striped_copy(full, s, r, shard, true, static_cast<cudaStream_t>(cuda_stream));
}

cdsp_status cdsp_striped_scatter(const cdsp_tensor* shard, int32_t s, int32_t r, cdsp_tensor* full,
                                 void* cuda_stream) {
    return striped_copy(full, s, r, const_cast<cdsp_tensor*>(shard), false, static_cast<cudaStream_t>(cuda_stream));
}

cdsp_status cdsp_zigzag_gather(const cdsp_tensor* full, int32_t s, int32_t r, cdsp_tensor* shard, void* cuda_stream) {
    return zigzag_copy(full, s, r, shard, true, static_cast<cudaStream_t>(cuda_stream));
}

cdsp_status cdsp_zigzag_scatter(const cdsp_tensor* shard, int32_t s, int32_t r, cdsp_tensor* full,
                                void* cuda_stream) {
    return zigzag_copy(full, s, r, const_cast<cdsp_tensor*>(shard), false, static_cast<cudaStream_t>(cuda_stream));
}

cdsp_status cdsp_zigzag_map_device(int64_t L, int32_t s, int32_t* tok_rank, int32_t* tok_slot, void* cuda_stream) {
    CDSP_REQUIRE(s == 1 || s == 2 || s == 4 || s == 8, CDSP_ERR_PLAN, "s=%d not in {1,2,4,8}", s);
    CDSP_REQUIRE(L >= 0 && L % (2 * s) == 0, CDSP_ERR_SHAPE, "L=%lld not a multiple of 2s", static_cast<long long>(L));
    return launch_zigzag_map(L, s, tok_rank, tok_slot, static_cast<cudaStream_t>(cuda_stream));
}

}  // extern "C"
