"""CPU oracle for the CDSP hot path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product path
(``paper_2511_06247_b200``) never imports it; the two share no code.

This module is argument marshalling (numpy <-> ctypes) around ``cdsp_oracle.c``, where
the arithmetic lives, each function citing the PAPER.md passage it writes out.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "cdsp_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

ORACLE_OK = 0
ORACLE_ERR_ARG = 1
ORACLE_ERR_PLAN = 4
ORACLE_ERR_RANGE = 5


def build(force: bool = False) -> str:
    """Compile cdsp_oracle.c with gcc (-O2, no fast-math, OpenMP over rows only)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fopenmp", "-fPIC", "-shared",
                               "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        P = ctypes.c_void_p
        i64, i32, dbl = ctypes.c_int64, ctypes.c_int32, ctypes.c_double
        _lib.oracle_attention.argtypes = [P, P, i64, P, P, P, i64, i32, i32, i32, dbl, P, P]
        _lib.oracle_causal_rows.argtypes = [P, P, P, i64, i32, i32, i32, dbl, P, i64, P, P]
        _lib.oracle_zigzag_map.argtypes = [i64, i32, P, P]
        _lib.oracle_plan_stores.argtypes = [i32, P, P, P, i32, P, P, i64, P, P]
        _lib.oracle_plan_stores_il.argtypes = [i32, P, P, P, P, i32, P, P, i64, P, P]
        _lib.oracle_striped_map.argtypes = [i64, i32, P, P]
        _lib.oracle_paged_write.argtypes = [P, P, i64, i32, i32, i32, i32, i32, P, i64, i64, P]
        _lib.oracle_lse_merge.argtypes = [i32, P, P, i64, i32, i32, P, P]
        for f in ("oracle_attention", "oracle_causal_rows", "oracle_zigzag_map", "oracle_striped_map",
                  "oracle_plan_stores", "oracle_plan_stores_il", "oracle_paged_write", "oracle_lse_merge",
                  "oracle_num_threads"):
            getattr(_lib, f).restype = ctypes.c_int
    return _lib


def num_threads() -> int:
    return int(lib().oracle_num_threads())


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _f32(a) -> np.ndarray:
    a = np.asarray(a)
    if a.dtype != np.float32:
        # every bf16 / fp32 input value is exactly representable in float32
        a = a.astype(np.float32)
    return np.ascontiguousarray(a)


class OracleError(RuntimeError):
    def __init__(self, rc: int, what: str):
        super().__init__(f"{what} returned {rc}")
        self.rc = rc


def _check(rc: int, what: str):
    if rc != ORACLE_OK:
        raise OracleError(rc, what)


def attention(q, qpos, k, v, kpos, scale: float):
    """Masked attention (visible iff kpos <= qpos).  q [nq,Hq,D], k/v [nk,Hkv,D].
    Returns (out [nq,Hq,D] f64, lse [Hq,nq] f64)."""
    q, k, v = _f32(q), _f32(k), _f32(v)
    qpos = np.ascontiguousarray(qpos, dtype=np.int64)
    kpos = np.ascontiguousarray(kpos, dtype=np.int64)
    nq, Hq, D = q.shape
    nk, Hkv, _ = k.shape
    out = np.empty((nq, Hq, D), np.float64)
    lse = np.empty((Hq, nq), np.float64)
    _check(lib().oracle_attention(_p(q), _p(qpos), nq, _p(k), _p(v), _p(kpos), nk,
                                  Hq, Hkv, D, float(scale), _p(out), _p(lse)), "oracle_attention")
    return out, lse


def causal_rows(q, k, v, scale: float, rows=None):
    """Causal attention over the whole unsharded prompt (q,k,v full [N,H,D]) for the
    query positions `rows` (None: all).  Returns (out [n,Hq,D], lse [Hq,n]) in f64."""
    q, k, v = _f32(q), _f32(k), _f32(v)
    N, Hq, D = q.shape
    Hkv = k.shape[1]
    if rows is None:
        n = N
        rp = None
    else:
        rows = np.ascontiguousarray(rows, dtype=np.int64)
        n = rows.shape[0]
        rp = _p(rows)
    out = np.empty((n, Hq, D), np.float64)
    lse = np.empty((Hq, n), np.float64)
    _check(lib().oracle_causal_rows(_p(q), _p(k), _p(v), N, Hq, Hkv, D, float(scale),
                                    rp, n, _p(out), _p(lse)), "oracle_causal_rows")
    return out, lse


def zigzag_map(L: int, s: int):
    """(tok_rank int32 [L], tok_slot int32 [L]) of P:75's zigzag partition."""
    tr = np.empty(L, np.int32)
    ts = np.empty(L, np.int32)
    _check(lib().oracle_zigzag_map(L, s, _p(tr), _p(ts)), "oracle_zigzag_map")
    return tr, ts


def striped_map(L: int, s: int):
    """(tok_rank int32 [L], tok_slot int32 [L]) of the striped (round-robin) partition."""
    tr = np.empty(L, np.int32)
    ts = np.empty(L, np.int32)
    _check(lib().oracle_striped_map(L, s, _p(tr), _p(ts)), "oracle_striped_map")
    return tr, ts


def rank_positions(L: int, s: int, C: int = 0, interleave: str = "zigzag"):
    """[s, 2m] int64 global positions of each ring rank's shard rows, derived from the
    oracle's zigzag (or striped) map (row tok_slot[t] of rank tok_rank[t] holds position C + t)."""
    tr, ts = (striped_map if interleave == "striped" else zigzag_map)(L, s)
    m = L // (2 * s)
    pos = np.full((s, 2 * m), -1, np.int64)
    pos[tr, ts] = C + np.arange(L, dtype=np.int64)
    return pos


def plan_stores(plan, upto: int):
    """Store state right before chunk `upto` computes (after its balancing).

    plan: list of (len, [ring-order instance ids]) or (len, ids, "striped" | "zigzag").
    Returns (store_n [s], store_pos list of int64 arrays, moves list of (src,dst,off,n))."""
    n_chunks = len(plan)
    lens = np.array([c[0] for c in plan], np.int64)
    sps = np.array([len(c[1]) for c in plan], np.int32)
    ranks = np.array([r for c in plan for r in c[1]], np.int32)
    il = np.array([1 if (len(c) > 2 and c[2] == "striped") else 0 for c in plan], np.int32)
    total = int(lens.sum())
    s = int(sps[upto])
    store_n = np.zeros(s, np.int64)
    stride = max(total, 1)
    store_pos = np.zeros((s, stride), np.int64)
    moves = np.zeros((8, 4), np.int64)
    nm = np.zeros(1, np.int32)
    _check(lib().oracle_plan_stores_il(n_chunks, _p(lens), _p(sps), _p(ranks), _p(il), upto, _p(store_n),
                                       _p(store_pos), stride, _p(moves), _p(nm)), "oracle_plan_stores")
    return (store_n, [store_pos[i, :store_n[i]].copy() for i in range(s)],
            [tuple(int(x) for x in moves[i]) for i in range(int(nm[0]))])


def paged_write(src: np.ndarray, pos, tp: int, block: int, block_table, dst_caches):
    """Write src [n,Hkv,D] (any dtype, byte copy) into dst_caches (list of tp arrays
    [num_blocks, block, Hkv/tp, D], same dtype), in place."""
    src = np.ascontiguousarray(src)
    pos = np.ascontiguousarray(pos, dtype=np.int64)
    bt = np.ascontiguousarray(block_table, dtype=np.int32)
    n, Hkv, D = src.shape
    assert len(dst_caches) == tp
    for d in dst_caches:
        assert d.flags["C_CONTIGUOUS"] and d.dtype == src.dtype
    num_blocks = dst_caches[0].shape[0]
    ptrs = (ctypes.c_void_p * tp)(*[d.ctypes.data for d in dst_caches])
    _check(lib().oracle_paged_write(_p(src), _p(pos), n, Hkv, D, src.dtype.itemsize, tp, block,
                                    _p(bt), bt.shape[0], num_blocks,
                                    ctypes.cast(ptrs, ctypes.c_void_p)), "oracle_paged_write")


def lse_merge(o_parts, lse_parts):
    """n-way merge: o_parts list of [T,H,D], lse_parts list of [H,T] -> (out, lse) f64."""
    n = len(o_parts)
    os_ = [np.ascontiguousarray(o, dtype=np.float64) for o in o_parts]
    ls_ = [np.ascontiguousarray(l, dtype=np.float64) for l in lse_parts]
    T, H, D = os_[0].shape
    out = np.empty((T, H, D), np.float64)
    lse = np.empty((H, T), np.float64)
    op = (ctypes.c_void_p * n)(*[o.ctypes.data for o in os_])
    lp = (ctypes.c_void_p * n)(*[l.ctypes.data for l in ls_])
    _check(lib().oracle_lse_merge(n, ctypes.cast(op, ctypes.c_void_p), ctypes.cast(lp, ctypes.c_void_p),
                                  T, H, D, _p(out), _p(lse)), "oracle_lse_merge")
    return out, lse
