// internal.h — launchers shared between the libcdsp.so translation units (not exported).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>

#include "cdsp.h"

namespace cdsp {

// One block-attention launch (see cdsp_attention_fwd / cdsp_attention_fwd_blocks in cdsp.h):
// the queries against nblk KV blocks (k[b], v[b], seg[b]; the query fields of every seg[b]
// are equal), walked in order with one softmax state per query row.
struct AttnArgs {
    const void* q = nullptr;
    int nblk = 1;
    const void* k[CDSP_MAX_SP] = {};
    const void* v[CDSP_MAX_SP] = {};
    cdsp_segments seg[CDSP_MAX_SP] = {};
    int32_t dtype = CDSP_BF16;
    int Hq = 0, Hkv = 0, D = 0;
    float scale = 0.f;   // softmax scale sigma
    int mode = CDSP_ATTN_ONLY;  // cdsp_attn_mode
    float* o_acc = nullptr;
    float* lse_acc = nullptr;
    void* out = nullptr;
    float* lse = nullptr;
    // launch as a programmatic dependent of the previous kernel in the stream (MID / LAST only:
    // the accumulator is touched after griddepcontrol.wait); internal ring chains and explicit
    // opt-in (CDSP_ATTN_PDL) only
    bool pdl = false;
    // arrival gating of blocks (bf16 kernel; see TcParams in attn_tc.cu); gate == NULL: none
    const uint32_t* gate = nullptr;
    uint32_t gate_target = 0, gate_mask = 0;
    int gate_ng = 1, gate_hpg = 1;
    int* gate_err = nullptr;
    int spare_sms = 0;  // leave at least this many SMs to other kernels (persistent bf16 grid)
    // an ONLY-mode multi-block launch may split its heavy units, merging them through o_acc /
    // lse_acc (their rows are scratch then)
    bool split_ok = false;
};

// Per-device kernel state (unit counters), allocated once; cdsp_comm_create calls it so the
// prefill path never allocates.
cdsp_status attention_device_init();

// KV tiles (128 keys) the bf16 kernel can list per launch (all blocks together).
int attention_tc_max_tiles(int D);
// TMA descriptor of a [rows, H, D] bf16 tensor: 128-byte swizzle, box = box_rows x 1 head x 64 d
// (zero fill out of bounds); defined in attn_tc.cu, used by the decode kernel
cdsp_status make_tile_map(CUtensorMap* m, const void* base, int64_t rows, int H, int D, int box_rows);

cdsp_status launch_attention_tc(const AttnArgs& a, cudaStream_t st);    // bf16, tcgen05/TMEM/TMA
cdsp_status launch_attention_simt(const AttnArgs& a, cudaStream_t st);  // fp32, FFMA

// n-way LSE merge.  parts[i] fp32 [T,H,D], lses[i] fp32 [H,T].
constexpr int kMaxMerge = 16;
cdsp_status launch_lse_merge(int n, const float* const* parts, const float* const* lses, int64_t T, int H,
                             int D, void* out, int32_t out_dtype, float* lse, cudaStream_t st);

// Row-segment copy: dst rows [dst_row0 + i] = src rows [src_row0 + i], i < n_rows, for up to
// two (src, dst) segment pairs; rows are `row_bytes` long (multiple of 16).
struct RowCopy {
    const void* src;
    void* dst;
    int64_t src_row0, dst_row0, n_rows;
    int64_t src_stride = 1, dst_stride = 1;  // row i: src_row0 + i src_stride -> dst_row0 + i dst_stride
};
cdsp_status launch_row_copy(const RowCopy* segs, int n_segs, int64_t row_bytes, cudaStream_t st);

// Store append: k/v rows + int32 positions (two contiguous position segments).
struct AppendArgs {
    const void* k_src;
    const void* v_src;
    void* k_dst;
    void* v_dst;
    int32_t* pos_dst;
    int64_t n_rows, row_bytes;
    int64_t len0, pos0, pos1;  // row i < len0 -> pos0 + i st, else pos1 + (i - len0) st
    int64_t pos_stride = 1;    // st: 1 zigzag, s striped
};
cdsp_status launch_store_append(const AppendArgs& a, cudaStream_t st);
// Store positions only: dst[i] = i < len0 ? pos0 + i st : pos1 + (i - len0) st.
cdsp_status launch_fill_positions(int32_t* dst, int64_t n, int64_t len0, int64_t pos0, int64_t pos1, int64_t pst,
                                  cudaStream_t st);

cdsp_status launch_zigzag_map(int64_t L, int s, int32_t* tok_rank, int32_t* tok_slot, cudaStream_t st);

// Paged-KV scatter (R15).
struct PagedArgs {
    const void* k;
    const void* v;
    int64_t n_tok;
    int Hkv, D, esize;
    int64_t len0, pos0, pos1;  // row -> position, as AppendArgs
    int64_t pos_stride;
    int tp, block_size;
    int64_t num_blocks, n_table;
    const int32_t* block_table;
    void* k_cache[8];
    void* v_cache[8];
    unsigned long long* bad_count;
    int seg_vec, seg_shift;  // set by the launcher: 16-B vectors per TP slice, log2 (or -1)
};
cdsp_status launch_paged_scatter(const PagedArgs& a, cudaStream_t st);

// Peer barrier: signal every listed peer, wait for each peer's matching signal.  remote[j] NULL:
// wait only; target[j] 0: signal only.
struct BarrierArgs {
    int n;
    unsigned long long* remote[8];  // peer j's flag slot for this instance (peer memory)
    unsigned long long* local[8];   // this instance's flag slot for peer j
    unsigned long long target[8];
    int* err;                       // host-mapped error word
};
cdsp_status launch_peer_barrier(const BarrierArgs& a, cudaStream_t st);

}  // namespace cdsp
