"""Thin ctypes binding of libcdsp.so (include/cdsp.h) — argument marshalling only.

Every step of the hot path runs in the library's CUDA kernels; torch is used for device
memory, streams and process groups.  There is no CPU fallback: if libcdsp.so is missing
or cannot load, every call raises.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np
import torch

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libcdsp.so")

CDSP_OK = 0
STATUS_NAMES = {0: "CDSP_OK", 1: "CDSP_ERR_INVALID", 2: "CDSP_ERR_SHAPE", 3: "CDSP_ERR_DTYPE",
                4: "CDSP_ERR_PLAN", 5: "CDSP_ERR_CAPACITY", 6: "CDSP_ERR_CUDA", 7: "CDSP_ERR_COMM",
                8: "CDSP_ERR_UNSUPPORTED"}
CDSP_F32, CDSP_BF16 = 0, 1
ATTN_ONLY, ATTN_FIRST, ATTN_MID, ATTN_LAST = 0, 1, 2, 3
ATTN_PDL = 0x100
RING_STEPWISE, RING_CONTROL, RING_GATE_FLAGS, RING_GATE_EVENTS = 1, 2, 4, 8
IPC_HANDLE_BYTES = 64

EXPORTED_SYMBOLS = (
    "cdsp_comm_create", "cdsp_comm_ipc_handle", "cdsp_comm_connect", "cdsp_comm_connect_local",
    "cdsp_comm_check", "cdsp_comm_destroy", "cdsp_kvstore_get", "cdsp_kvstore_reset",
    "cdsp_plan_capacity", "cdsp_plan_partition", "cdsp_prefill_chunk", "cdsp_lse_merge", "cdsp_kv_transfer_to_decode",
    "cdsp_attention_fwd", "cdsp_zigzag_gather", "cdsp_zigzag_scatter", "cdsp_zigzag_map_device",
    "cdsp_kv_transfer_errors", "cdsp_last_error", "cdsp_abi_version", "cdsp_comm_profile",
    "cdsp_comm_profile_read", "cdsp_decode_workspace_bytes", "cdsp_decode_attention", "cdsp_comm_profile_ring",
    "cdsp_comm_create_layers", "cdsp_kvstore_get_layer", "cdsp_prefill_chunk_layer",
    "cdsp_striped_gather", "cdsp_striped_scatter", "cdsp_fit_latency_model", "cdsp_schedule_prefill",
    "cdsp_comm_reserve", "cdsp_comm_set_ring_options", "cdsp_attention_fwd_blocks", "cdsp_prefill_chunk_transfer",
    "cdsp_decode_attention_batch",
)


class CdspError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


# ---- C structs (mirror include/cdsp.h) ---------------------------------------------------
class Tensor(ctypes.Structure):
    _fields_ = [("ptr", ctypes.c_void_p), ("dtype", ctypes.c_int32), ("T", ctypes.c_int64),
                ("H", ctypes.c_int64), ("D", ctypes.c_int64)]


class Chunk(ctypes.Structure):
    _fields_ = [("len", ctypes.c_int64), ("sp", ctypes.c_int32), ("interleave", ctypes.c_int32),
                ("ranks", ctypes.POINTER(ctypes.c_int32))]


class PlanC(ctypes.Structure):
    _fields_ = [("n_chunks", ctypes.c_int32), ("chunks", ctypes.POINTER(Chunk))]


class Move(ctypes.Structure):
    _fields_ = [("src", ctypes.c_int32), ("dst", ctypes.c_int32), ("src_off", ctypes.c_int64),
                ("n_tok", ctypes.c_int64)]


class KvStoreC(ctypes.Structure):
    _fields_ = [("k", Tensor), ("v", Tensor), ("pos", ctypes.c_void_p), ("n", ctypes.c_int64),
                ("cap", ctypes.c_int64)]


class SpGroupC(ctypes.Structure):
    _fields_ = [("comm", ctypes.c_void_p), ("plan", ctypes.POINTER(PlanC)), ("chunk", ctypes.c_int32)]


class DecodeTargetC(ctypes.Structure):
    _fields_ = [("tp", ctypes.c_int32), ("block_size", ctypes.c_int32), ("num_blocks", ctypes.c_int64),
                ("k_cache", ctypes.POINTER(ctypes.c_void_p)), ("v_cache", ctypes.POINTER(ctypes.c_void_p)),
                ("block_table", ctypes.c_void_p), ("n_table", ctypes.c_int64)]


class Segments(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int64) for n in ("nq", "q_len0", "q_pos0", "q_pos1", "nkv", "kv_hist",
                                              "kv_len0", "kv_pos0", "kv_pos1", "pos_stride")]


class LatencyModel(ctypes.Structure):
    _fields_ = [("a", ctypes.c_double), ("b", ctypes.c_double), ("c", ctypes.c_double), ("d", ctypes.c_double)]


MAX_CHUNKS = 8


class ScheduleC(ctypes.Structure):
    _fields_ = [("n_chunks", ctypes.c_int32), ("len", ctypes.c_int64 * MAX_CHUNKS), ("sp", ctypes.c_int32 * MAX_CHUNKS),
                ("ranks", (ctypes.c_int32 * 8) * MAX_CHUNKS), ("ttft", ctypes.c_double)]


_lib = None


def lib():
    """Load libcdsp.so (raises if it is missing: the product path has no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing; run paper_2511_06247_b200/build.py "
                              "(or __graft_entry__.build())")
        L = ctypes.CDLL(LIB_PATH)
        P, i32, i64, f32 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_float
        sig = {
            "cdsp_comm_create": [ctypes.POINTER(P), i32, i32, i32, i64, i32, i32, i32],
            "cdsp_comm_create_layers": [ctypes.POINTER(P), i32, i32, i32, i64, i32, i32, i32, i32],
            "cdsp_kvstore_get_layer": [P, i32, ctypes.POINTER(KvStoreC)],
            "cdsp_prefill_chunk_layer": [ctypes.POINTER(Tensor)] * 3 + [ctypes.POINTER(KvStoreC),
                                                                        ctypes.POINTER(SpGroupC), i32, f32,
                                                                        ctypes.POINTER(Tensor), P, P],
            "cdsp_comm_reserve": [P, i64, i32],
            "cdsp_comm_set_ring_options": [P, i32],
            "cdsp_attention_fwd_blocks": [ctypes.POINTER(Tensor), i32, ctypes.POINTER(ctypes.POINTER(Tensor)),
                                          ctypes.POINTER(ctypes.POINTER(Tensor)), ctypes.POINTER(Segments), f32, i32,
                                          P, P, ctypes.POINTER(Tensor), P, P],
            "cdsp_comm_ipc_handle": [P, P],
            "cdsp_comm_connect": [P, P],
            "cdsp_comm_connect_local": [ctypes.POINTER(P), i32],
            "cdsp_comm_check": [P],
            "cdsp_comm_destroy": [P],
            "cdsp_kvstore_get": [P, ctypes.POINTER(KvStoreC)],
            "cdsp_kvstore_reset": [P, P],
            "cdsp_plan_capacity": [ctypes.POINTER(PlanC), ctypes.POINTER(i64)],
            "cdsp_plan_partition": [ctypes.POINTER(PlanC), i32, P, P, P, P, P],
            "cdsp_prefill_chunk": [ctypes.POINTER(Tensor)] * 3 + [ctypes.POINTER(KvStoreC),
                                                                  ctypes.POINTER(SpGroupC), f32,
                                                                  ctypes.POINTER(Tensor), P, P],
            "cdsp_prefill_chunk_transfer": [ctypes.POINTER(Tensor)] * 3 + [ctypes.POINTER(KvStoreC),
                                                                           ctypes.POINTER(SpGroupC), f32,
                                                                           ctypes.POINTER(Tensor), P,
                                                                           ctypes.POINTER(DecodeTargetC), P],
            "cdsp_lse_merge": [i32, ctypes.POINTER(ctypes.POINTER(Tensor)), ctypes.POINTER(P),
                               ctypes.POINTER(Tensor), P, P],
            "cdsp_kv_transfer_to_decode": [ctypes.POINTER(Tensor), ctypes.POINTER(Tensor),
                                           ctypes.POINTER(SpGroupC), ctypes.POINTER(DecodeTargetC), P],
            "cdsp_attention_fwd": [ctypes.POINTER(Tensor)] * 3 + [ctypes.POINTER(Segments), f32, i32, P, P,
                                                                  ctypes.POINTER(Tensor), P, P],
            "cdsp_zigzag_gather": [ctypes.POINTER(Tensor), i32, i32, ctypes.POINTER(Tensor), P],
            "cdsp_zigzag_scatter": [ctypes.POINTER(Tensor), i32, i32, ctypes.POINTER(Tensor), P],
            "cdsp_striped_gather": [ctypes.POINTER(Tensor), i32, i32, ctypes.POINTER(Tensor), P],
            "cdsp_striped_scatter": [ctypes.POINTER(Tensor), i32, i32, ctypes.POINTER(Tensor), P],
            "cdsp_zigzag_map_device": [i64, i32, P, P, P],
            "cdsp_kv_transfer_errors": [P, P, ctypes.POINTER(i64)],
            "cdsp_comm_profile": [P, i32],
            "cdsp_comm_profile_read": [P, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(i32)],
            "cdsp_decode_workspace_bytes": [i32, i32, i32, ctypes.POINTER(ctypes.c_size_t)],
            "cdsp_fit_latency_model": [i32, P, P, P, ctypes.POINTER(LatencyModel)],
            "cdsp_schedule_prefill": [i64, i32, P, i32, i32, P, P, ctypes.c_double, i64, ctypes.POINTER(ScheduleC)],
            "cdsp_comm_profile_ring": [P, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double),
                                       ctypes.POINTER(i64), ctypes.POINTER(i32)],
            "cdsp_decode_attention": [ctypes.POINTER(Tensor), ctypes.POINTER(DecodeTargetC), i32, i32, i64, f32,
                                      ctypes.POINTER(Tensor), P, P, ctypes.c_size_t, P],
            "cdsp_decode_attention_batch": [ctypes.POINTER(Tensor), ctypes.POINTER(DecodeTargetC), i32, i32, i32, P,
                                            f32, ctypes.POINTER(Tensor), P, P, ctypes.c_size_t, P],
        }
        for name, args in sig.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = ctypes.c_int
        L.cdsp_last_error.restype = ctypes.c_char_p
        L.cdsp_last_error.argtypes = []
        L.cdsp_abi_version.restype = ctypes.c_int32
        _lib = L
    return _lib


def _check(status: int):
    if status != CDSP_OK:
        raise CdspError(status, lib().cdsp_last_error().decode())


def _dtype_code(t: torch.dtype) -> int:
    if t == torch.float32:
        return CDSP_F32
    if t == torch.bfloat16:
        return CDSP_BF16
    raise CdspError(3, f"unsupported dtype {t}")


def as_tensor(x: torch.Tensor) -> Tensor:
    """[T, H, D] contiguous torch tensor -> cdsp_tensor (no copy)."""
    if x.dim() != 3:
        raise CdspError(2, f"expected a [T,H,D] tensor, got shape {tuple(x.shape)}")
    if not x.is_contiguous():
        raise CdspError(1, "tensor must be contiguous")
    return Tensor(x.data_ptr(), _dtype_code(x.dtype), x.shape[0], x.shape[1], x.shape[2])


def _stream(stream) -> ctypes.c_void_p:
    if stream is None:
        stream = torch.cuda.current_stream()
    if isinstance(stream, torch.cuda.Stream):
        return ctypes.c_void_p(stream.cuda_stream)
    return ctypes.c_void_p(int(stream))


def _ptr(x: Optional[torch.Tensor]):
    return ctypes.c_void_p(x.data_ptr() if x is not None else 0)


# ---- plan ----------------------------------------------------------------------------------
INTERLEAVE = {"zigzag": 0, "striped": 1}


class Plan:
    """CDSP plan A = [(token count, ring-order instance group[, "zigzag" | "striped"])] (
    interleave per chunk, "striped/zigzag", default zigzag)."""

    def __init__(self, chunks: Sequence[tuple]):
        self.chunks = [(int(c[0]), [int(r) for r in c[1]]) for c in chunks]
        self.interleave = [c[2] if len(c) > 2 else "zigzag" for c in chunks]
        self._rank_arrays = [(ctypes.c_int32 * len(r))(*r) for _, r in self.chunks]
        arr = (Chunk * len(self.chunks))()
        for i, (L, r) in enumerate(self.chunks):
            arr[i] = Chunk(L, len(r), INTERLEAVE[self.interleave[i]],
                           ctypes.cast(self._rank_arrays[i], ctypes.POINTER(ctypes.c_int32)))
        self._arr = arr
        self.c = PlanC(len(self.chunks), ctypes.cast(arr, ctypes.POINTER(Chunk)))

    def chunk_start(self, c: int) -> int:
        return sum(L for L, _ in self.chunks[:c])

    def __len__(self):
        return len(self.chunks)


def fit_latency_model(C, L, T):
    """cdsp_fit_latency_model: Eq. (1) coefficients (a, b, c, d) from samples."""
    C, L, T = (np.ascontiguousarray(x, dtype=np.float64) for x in (C, L, T))
    out = LatencyModel()
    _check(lib().cdsp_fit_latency_model(len(T), C.ctypes.data, L.ctypes.data, T.ctypes.data, ctypes.byref(out)))
    return (out.a, out.b, out.c, out.d)


def schedule_prefill(L: int, queue, node_size: int, models: dict, improvement_rate: float, granule: int):
    """cdsp_schedule_prefill: -> ([(len, ring-order ranks)], ttft).  models: {s: (a, b, c, d)}."""
    q = np.ascontiguousarray(queue, dtype=np.float64)
    sizes = sorted(models)
    sz = np.array(sizes, np.int32)
    ms = (LatencyModel * len(sizes))(*[LatencyModel(*models[s]) for s in sizes])
    out = ScheduleC()
    _check(lib().cdsp_schedule_prefill(int(L), len(q), q.ctypes.data, node_size, len(sizes), sz.ctypes.data,
                                       ctypes.cast(ms, ctypes.c_void_p), float(improvement_rate), int(granule),
                                       ctypes.byref(out)))
    plan = [(int(out.len[c]), [int(out.ranks[c][r]) for r in range(out.sp[c])]) for c in range(out.n_chunks)]
    return plan, float(out.ttft)


def plan_capacity(plan: Plan) -> int:
    """Store rows per instance the plan needs (largest history + shard of any ring rank)."""
    n = ctypes.c_int64(0)
    _check(lib().cdsp_plan_capacity(ctypes.byref(plan.c), ctypes.byref(n)))
    return int(n.value)


def plan_partition(plan: Plan, c: int):
    """-> (tok_rank int32 [L], tok_slot int32 [L], rank_pos int64 [s, 2m], moves list)."""
    if not 0 <= c < len(plan.chunks):
        _check(lib().cdsp_plan_partition(ctypes.byref(plan.c), c, None, None, None, None, None))
    L, ranks = plan.chunks[c]
    s = len(ranks)
    tr = np.empty(L, np.int32)
    ts = np.empty(L, np.int32)
    rp = np.empty((s, L // s), np.int64)
    mv = (Move * 8)()
    nm = ctypes.c_int32(0)
    _check(lib().cdsp_plan_partition(ctypes.byref(plan.c), c, tr.ctypes.data, ts.ctypes.data, rp.ctypes.data,
                                     ctypes.cast(mv, ctypes.c_void_p), ctypes.byref(nm)))
    moves = [(mv[i].src, mv[i].dst, mv[i].src_off, mv[i].n_tok) for i in range(nm.value)]
    return tr, ts, rp, moves


# ---- communicator ----------------------------------------------------------------------------
@dataclass
class KvStore:
    """View of a communicator's KV store (cdsp_kvstore)."""
    c: KvStoreC
    k: torch.Tensor
    v: torch.Tensor
    pos: torch.Tensor

    @property
    def n(self) -> int:
        return int(self.c.n)


class Comm:
    def __init__(self, rank: int, world: int, device: int, store_cap_tokens: int, Hkv: int, D: int,
                 dtype: torch.dtype = torch.bfloat16, n_layers: int = 1, max_q_rows: int = 0, max_hq: int = 0):
        """cdsp_comm_create_layers (+ cdsp_comm_reserve(max_q_rows, max_hq) when both are given)."""
        self.rank, self.world, self.device = rank, world, device
        self.Hkv, self.D, self.dtype, self.n_layers = Hkv, D, dtype, n_layers
        h = ctypes.c_void_p()
        _check(lib().cdsp_comm_create_layers(ctypes.byref(h), rank, world, device, int(store_cap_tokens), n_layers,
                                             Hkv, D, _dtype_code(dtype)))
        self.h = h
        self.cap = int(store_cap_tokens)
        self._stores = {}
        if max_q_rows and max_hq:
            self.reserve(max_q_rows, max_hq)

    def reserve(self, max_q_rows: int, max_hq: int):
        """cdsp_comm_reserve: fp32 merge accumulators for multi-launch rings."""
        _check(lib().cdsp_comm_reserve(self.h, int(max_q_rows), int(max_hq)))

    def set_ring_options(self, options: int):
        """cdsp_comm_set_ring_options (RING_* bits)."""
        _check(lib().cdsp_comm_set_ring_options(self.h, int(options)))

    def ipc_handle(self) -> bytes:
        buf = ctypes.create_string_buffer(IPC_HANDLE_BYTES)
        _check(lib().cdsp_comm_ipc_handle(self.h, buf))
        return buf.raw

    def connect(self, handles: Sequence[bytes]):
        blob = b"".join(handles)
        _check(lib().cdsp_comm_connect(self.h, blob))

    def connect_process_group(self, group=None):
        """Exchange IPC handles over torch.distributed (plumbing) and open the peers."""
        from .dist_utils import exchange_bytes
        self.connect(exchange_bytes(self.ipc_handle(), group))

    def check(self):
        _check(lib().cdsp_comm_check(self.h))

    def profile(self, enable: bool = True):
        """Bracket every block-attention launch of this instance with CUDA events."""
        _check(lib().cdsp_comm_profile(self.h, 1 if enable else 0))

    def profile_read(self):
        """-> (summed attention kernel ms, number of launches) since the last read."""
        ms = ctypes.c_double(0.0)
        n = ctypes.c_int32(0)
        _check(lib().cdsp_comm_profile_read(self.h, ctypes.byref(ms), ctypes.byref(n)))
        return float(ms.value), int(n.value)

    def profile_ring(self):
        """-> (pull ms, exposed ms, bytes, pulls) of the ring since the last read (see cdsp.h)."""
        cp, ex = ctypes.c_double(0.0), ctypes.c_double(0.0)
        by, n = ctypes.c_int64(0), ctypes.c_int32(0)
        _check(lib().cdsp_comm_profile_ring(self.h, ctypes.byref(cp), ctypes.byref(ex), ctypes.byref(by),
                                            ctypes.byref(n)))
        return float(cp.value), float(ex.value), int(by.value), int(n.value)

    def kvstore(self, layer: int = 0) -> KvStore:
        c = KvStoreC()
        _check(lib().cdsp_kvstore_get_layer(self.h, layer, ctypes.byref(c)))
        st = self._stores.get(layer)
        if st is None:
            st = self._stores[layer] = _wrap_store(c, self)
        st.c = c
        return st

    def reset(self, stream=None):
        _check(lib().cdsp_kvstore_reset(self.h, _stream(stream)))

    def close(self):
        if self.h:
            _check(lib().cdsp_comm_destroy(self.h))
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _wrap_store(c: KvStoreC, comm: Comm) -> KvStore:
    """Torch views of the comm-owned store memory (for inspection in tests)."""
    cap, H, D = int(c.cap), comm.Hkv, comm.D
    es = 2 if comm.dtype == torch.bfloat16 else 4
    k = _device_view(c.k.ptr, cap * H * D * es, comm.device).view(comm.dtype).view(cap, H, D)
    v = _device_view(c.v.ptr, cap * H * D * es, comm.device).view(comm.dtype).view(cap, H, D)
    pos = _device_view(c.pos, cap * 4, comm.device).view(torch.int32)
    return KvStore(c, k, v, pos)


def _device_view(ptr: int, nbytes: int, device: int) -> torch.Tensor:
    """A uint8 torch tensor aliasing library-owned device memory (no ownership)."""
    class _CAI:
        __cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (int(ptr), False),
                                    "version": 3, "strides": None}
    with torch.cuda.device(device):
        return torch.as_tensor(_CAI(), device=f"cuda:{device}")


def connect_local(comms: Sequence[Comm]):
    arr = (ctypes.c_void_p * len(comms))(*[c.h.value for c in comms])
    _check(lib().cdsp_comm_connect_local(arr, len(comms)))


class SpGroup:
    def __init__(self, comm: Comm, plan: Plan, chunk: int):
        self.comm, self.plan, self.chunk = comm, plan, chunk
        self.c = SpGroupC(comm.h, ctypes.pointer(plan.c), chunk)


# ---- the four calls ----------------------------------------------------------------------------
def prefill_chunk(q, k, v, prev_kv: KvStore, sp_group: SpGroup, softmax_scale: float = 0.0,
                  out: Optional[torch.Tensor] = None, lse: Optional[torch.Tensor] = None, stream=None,
                  layer: Optional[int] = None):
    """cdsp_prefill_chunk (or cdsp_prefill_chunk_layer when `layer` is given): this rank's zigzag
    shard q/k/v [2m,H,D] -> out [2m,Hq,D] (+ lse [Hq,2m])."""
    if out is None:
        out = torch.empty_like(q)
    tq, tk, tv, to = as_tensor(q), as_tensor(k), as_tensor(v), as_tensor(out)
    if layer is None:
        _check(lib().cdsp_prefill_chunk(ctypes.byref(tq), ctypes.byref(tk), ctypes.byref(tv),
                                        ctypes.byref(prev_kv.c), ctypes.byref(sp_group.c), float(softmax_scale),
                                        ctypes.byref(to), _ptr(lse), _stream(stream)))
    else:
        _check(lib().cdsp_prefill_chunk_layer(ctypes.byref(tq), ctypes.byref(tk), ctypes.byref(tv),
                                              ctypes.byref(prev_kv.c), ctypes.byref(sp_group.c), int(layer),
                                              float(softmax_scale), ctypes.byref(to), _ptr(lse), _stream(stream)))
    return out


def prefill_chunk_transfer(q, k, v, prev_kv: KvStore, sp_group: SpGroup, dst: "DecodeTarget",
                           softmax_scale: float = 0.0, out: Optional[torch.Tensor] = None,
                           lse: Optional[torch.Tensor] = None, stream=None):
    """cdsp_prefill_chunk_transfer: prefill_chunk + kv_transfer_to_decode of the same shard (the
    transfer fused into the attention launch where the library can)."""
    if out is None:
        out = torch.empty_like(q)
    tq, tk, tv, to = as_tensor(q), as_tensor(k), as_tensor(v), as_tensor(out)
    _check(lib().cdsp_prefill_chunk_transfer(ctypes.byref(tq), ctypes.byref(tk), ctypes.byref(tv),
                                             ctypes.byref(prev_kv.c), ctypes.byref(sp_group.c), float(softmax_scale),
                                             ctypes.byref(to), _ptr(lse), ctypes.byref(dst.c), _stream(stream)))
    return out


def lse_merge(o_parts: Sequence[torch.Tensor], lse_parts: Sequence[torch.Tensor], out: torch.Tensor,
              lse: Optional[torch.Tensor] = None, stream=None):
    n = len(o_parts)
    ts = [as_tensor(o) for o in o_parts]
    tp = (ctypes.POINTER(Tensor) * n)(*[ctypes.pointer(t) for t in ts])
    lp = (ctypes.c_void_p * n)(*[l.data_ptr() for l in lse_parts])
    to = as_tensor(out)
    _check(lib().cdsp_lse_merge(n, tp, lp, ctypes.byref(to), _ptr(lse), _stream(stream)))
    return out


class DecodeTarget:
    """Decode paged KV caches (R15): tp lists of [num_blocks, block, Hkv/tp, D] tensors."""

    def __init__(self, k_caches: Sequence[torch.Tensor], v_caches: Sequence[torch.Tensor], block_size: int,
                 block_table: torch.Tensor):
        self.k_caches, self.v_caches, self.block_table = list(k_caches), list(v_caches), block_table
        tp = len(self.k_caches)
        self._k = (ctypes.c_void_p * tp)(*[t.data_ptr() for t in self.k_caches])
        self._v = (ctypes.c_void_p * tp)(*[t.data_ptr() for t in self.v_caches])
        self.c = DecodeTargetC(tp, block_size, self.k_caches[0].shape[0],
                               ctypes.cast(self._k, ctypes.POINTER(ctypes.c_void_p)),
                               ctypes.cast(self._v, ctypes.POINTER(ctypes.c_void_p)),
                               block_table.data_ptr(), block_table.numel())


def kv_transfer_to_decode(k, v, sp_group: SpGroup, dst: DecodeTarget, stream=None):
    tk, tv = as_tensor(k), as_tensor(v)
    _check(lib().cdsp_kv_transfer_to_decode(ctypes.byref(tk), ctypes.byref(tv), ctypes.byref(sp_group.c),
                                            ctypes.byref(dst.c), _stream(stream)))


def decode_workspace_bytes(hq_local: int, hkv_local: int, D: int) -> int:
    n = ctypes.c_size_t(0)
    _check(lib().cdsp_decode_workspace_bytes(hq_local, hkv_local, D, ctypes.byref(n)))
    return int(n.value)


def decode_workspace(hq_local: int, hkv_local: int, D: int, device="cuda") -> torch.Tensor:
    """Zero-filled workspace for cdsp_decode_attention (torch's caching allocator aligns to 512 B)."""
    return torch.zeros(decode_workspace_bytes(hq_local, hkv_local, D), dtype=torch.uint8, device=device)


def decode_attention(q, cache: DecodeTarget, t: int, hkv_local: int, n_ctx: int, softmax_scale: float = 0.0,
                     out=None, lse=None, workspace=None, stream=None):
    """Decode step on decode TP rank t over its paged cache: q [1, Hq_t, D] -> (out, lse [Hq_t])."""
    Hq_t, D = q.shape[1], q.shape[2]
    out = out if out is not None else torch.empty_like(q)
    if workspace is None:
        workspace = decode_workspace(Hq_t, hkv_local, D, q.device)
    tq, to = as_tensor(q), as_tensor(out)
    _check(lib().cdsp_decode_attention(ctypes.byref(tq), ctypes.byref(cache.c), t, hkv_local, n_ctx, softmax_scale,
                                       ctypes.byref(to), _ptr(lse), workspace.data_ptr(), workspace.numel(),
                                       _stream(stream)))
    return out, lse


def decode_attention_batch(q, cache: DecodeTarget, t: int, hkv_local: int, ctx_lens: Sequence[int],
                           softmax_scale: float = 0.0, out=None, lse=None, workspace=None, stream=None):
    """Decode step for a batch on decode TP rank t: q [batch, Hq_t, D], request b over row b of
    cache.block_table ([batch, pages]) up to ctx_lens[b] (host lengths) -> (out, lse [batch, Hq_t])."""
    batch, Hq_t, D = q.shape
    lens = (ctypes.c_int32 * batch)(*[int(x) for x in ctx_lens])
    out = out if out is not None else torch.empty_like(q)
    if workspace is None:
        workspace = decode_workspace(batch * Hq_t, batch * hkv_local, D, q.device)
    tq, to = as_tensor(q), as_tensor(out)
    _check(lib().cdsp_decode_attention_batch(ctypes.byref(tq), ctypes.byref(cache.c), t, hkv_local, batch,
                                             lens, softmax_scale, ctypes.byref(to),
                                             _ptr(lse), workspace.data_ptr(), workspace.numel(), _stream(stream)))
    return out, lse


def kv_transfer_errors(comm: Comm, stream=None) -> int:
    n = ctypes.c_int64(0)
    _check(lib().cdsp_kv_transfer_errors(comm.h, _stream(stream), ctypes.byref(n)))
    return int(n.value)


# ---- building blocks ------------------------------------------------------------------------------
def segments(nq, q_len0, q_pos0, q_pos1, nkv, kv_hist, kv_len0, kv_pos0, kv_pos1, pos_stride=1) -> Segments:
    return Segments(nq, q_len0, q_pos0, q_pos1, nkv, kv_hist, kv_len0, kv_pos0, kv_pos1, pos_stride)


def causal_segments(nq: int, nkv: int, q_pos0: int = 0, kv_hist: int = 0) -> Segments:
    """Contiguous queries at q_pos0.. over kv_hist history rows + contiguous keys at 0.."""
    return Segments(nq, nq, q_pos0, 0, nkv, kv_hist, nkv - kv_hist, 0, 0, 1)


def attention_fwd(q, k, v, seg: Segments, softmax_scale: float = 0.0, mode: int = ATTN_ONLY,
                  o_acc=None, lse_acc=None, out=None, lse=None, stream=None):
    tq, tk, tv = as_tensor(q), as_tensor(k), as_tensor(v)
    to = as_tensor(out) if out is not None else None
    _check(lib().cdsp_attention_fwd(ctypes.byref(tq), ctypes.byref(tk), ctypes.byref(tv), ctypes.byref(seg),
                                    float(softmax_scale), mode, _ptr(o_acc), _ptr(lse_acc),
                                    ctypes.byref(to) if to is not None else None, _ptr(lse), _stream(stream)))
    return out


def attention_fwd_blocks(q, ks, vs, segs, softmax_scale: float = 0.0, mode: int = ATTN_ONLY,
                         o_acc=None, lse_acc=None, out=None, lse=None, stream=None):
    """cdsp_attention_fwd_blocks: q against the union of KV blocks (ks[b], vs[b], segs[b]) in one launch."""
    n = len(ks)
    tq = as_tensor(q)
    tk = [as_tensor(x) for x in ks]
    tv = [as_tensor(x) for x in vs]
    pk = (ctypes.POINTER(Tensor) * n)(*[ctypes.pointer(t) for t in tk])
    pv = (ctypes.POINTER(Tensor) * n)(*[ctypes.pointer(t) for t in tv])
    sg = (Segments * n)(*segs)
    to = as_tensor(out) if out is not None else None
    _check(lib().cdsp_attention_fwd_blocks(ctypes.byref(tq), n, pk, pv, sg, float(softmax_scale), mode,
                                           _ptr(o_acc), _ptr(lse_acc), ctypes.byref(to) if to is not None else None,
                                           _ptr(lse), _stream(stream)))
    return out


def zigzag_gather(full, s: int, r: int, shard=None, stream=None):
    if shard is None:
        shard = torch.empty((full.shape[0] // s,) + tuple(full.shape[1:]), dtype=full.dtype, device=full.device)
    tf, ts = as_tensor(full), as_tensor(shard)
    _check(lib().cdsp_zigzag_gather(ctypes.byref(tf), s, r, ctypes.byref(ts), _stream(stream)))
    return shard


def striped_gather(full, s: int, r: int, shard=None, stream=None):
    if shard is None:
        shard = torch.empty((full.shape[0] // s,) + tuple(full.shape[1:]), dtype=full.dtype, device=full.device)
    tf, ts = as_tensor(full), as_tensor(shard)
    _check(lib().cdsp_striped_gather(ctypes.byref(tf), s, r, ctypes.byref(ts), _stream(stream)))
    return shard


def striped_scatter(shard, s: int, r: int, full, stream=None):
    ts, tf = as_tensor(shard), as_tensor(full)
    _check(lib().cdsp_striped_scatter(ctypes.byref(ts), s, r, ctypes.byref(tf), _stream(stream)))
    return full


def shard_gather(full, s: int, r: int, interleave: str = "zigzag", shard=None, stream=None):
    """This ring rank's shard of a chunk under the chunk's interleave."""
    f = striped_gather if interleave == "striped" else zigzag_gather
    return f(full, s, r, shard, stream)


def shard_scatter(shard, s: int, r: int, full, interleave: str = "zigzag", stream=None):
    f = striped_scatter if interleave == "striped" else zigzag_scatter
    return f(shard, s, r, full, stream)


def zigzag_scatter(shard, s: int, r: int, full, stream=None):
    ts, tf = as_tensor(shard), as_tensor(full)
    _check(lib().cdsp_zigzag_scatter(ctypes.byref(ts), s, r, ctypes.byref(tf), _stream(stream)))
    return full


def zigzag_map_device(L: int, s: int, device="cuda", stream=None):
    tr = torch.empty(L, dtype=torch.int32, device=device)
    ts = torch.empty(L, dtype=torch.int32, device=device)
    _check(lib().cdsp_zigzag_map_device(L, s, _ptr(tr), _ptr(ts), _stream(stream)))
    return tr, ts


def abi_version() -> int:
    return int(lib().cdsp_abi_version())
