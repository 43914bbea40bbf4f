"""Drivers that run a whole CDSP plan through the C ABI.

``run_plan_loopback``: every instance of the plan is a virtual rank on THIS GPU, each with
its own communicator and stream (cdsp_comm_connect_local).  The library calls only enqueue
work, so one host thread issues all ranks' calls in turn; the device-side peer barriers and
copy-engine pulls are the same code the multi-process path runs over NVLink.

``run_plan_distributed``: one process per GPU (torch.distributed for the IPC handle
exchange only); this process executes the chunks whose group contains its rank.

Input sharding (cdsp_zigzag_gather / cdsp_striped_gather, per the chunk's interleave) and
output reassembly (cdsp_zigzag_scatter / cdsp_striped_scatter) use the
library's kernels; the LSE reassembly for tests is harness code (index_copy).
"""
from __future__ import annotations

from typing import List, Optional, Sequence

import torch

from . import api


def _rank_lse_index(plan: api.Plan, c: int, r: int, device) -> torch.Tensor:
    _, _, rank_pos, _ = api.plan_partition(plan, c)
    return torch.as_tensor(rank_pos[r], device=device)


def max_shard_rows(plan: api.Plan) -> int:
    """Largest query shard 2m = L / s of the plan (the accumulator rows a multi-launch ring needs)."""
    return max(L // len(ranks) for L, ranks in plan.chunks)


def make_loopback_comms(plan: api.Plan, Hkv: int, D: int, dtype, device: int = 0, cap: Optional[int] = None,
                        Hq: Optional[int] = None):
    """One communicator per instance of the plan on `device`, linked as a loopback group.  With Hq
    given, each reserves fp32 accumulators for the plan's largest shard (multi-launch rings:
    fp32, oversized bf16 blocks, RING_STEPWISE)."""
    world = max(r for _, ranks in plan.chunks for r in ranks) + 1
    cap = cap or api.plan_capacity(plan)
    rows = max_shard_rows(plan) if Hq else 0
    comms = [api.Comm(i, world, device, cap, Hkv, D, dtype, max_q_rows=rows, max_hq=Hq or 0) for i in range(world)]
    if world > 1:
        api.connect_local(comms)
    return comms


def run_plan_loopback(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, plan: api.Plan,
                      softmax_scale: float = 0.0, comms: Optional[List[api.Comm]] = None,
                      streams: Optional[Sequence[torch.cuda.Stream]] = None, want_lse: bool = True,
                      shards=None, out_shards=None):
    """Full-prompt q [N,Hq,D], k/v [N,Hkv,D] on one device -> (out [N,Hq,D], lse [Hq,N] or None).

    ``shards`` (optional, reused across calls): per chunk, per ring rank, (q, k, v) shards
    prepared by :func:`prepare_shards`."""
    device = q.device
    N, Hq, D = q.shape
    Hkv = k.shape[1]
    assert sum(L for L, _ in plan.chunks) == N, "plan does not cover the prompt"
    if comms is None:
        comms = make_loopback_comms(plan, Hkv, D, q.dtype, device.index or 0, Hq=Hq)
    world = len(comms)
    if streams is None:
        streams = [torch.cuda.Stream(device=device) for _ in range(world)]
    cur = torch.cuda.current_stream(device)
    for s in streams:
        s.wait_stream(cur)
    for cm in comms:
        cm.reset(cur)
    if shards is None:
        shards = prepare_shards(q, k, v, plan, streams=None)
        for s in streams:
            s.wait_stream(cur)
    out = torch.empty_like(q)
    lse = torch.empty((Hq, N), dtype=torch.float32, device=device) if want_lse else None
    outs = out_shards if out_shards is not None else alloc_out_shards(plan, Hq, D, q.dtype, device, want_lse)
    for c, (L, ranks) in enumerate(plan.chunks):
        C = plan.chunk_start(c)
        for r, inst in enumerate(ranks):
            qs, ks, vs = shards[c][r]
            o_r, l_r = outs[c][r]
            api.prefill_chunk(qs, ks, vs, comms[inst].kvstore(), api.SpGroup(comms[inst], plan, c),
                              softmax_scale, o_r, l_r, stream=streams[inst])
        for r, inst in enumerate(ranks):
            with torch.cuda.stream(streams[inst]):
                o_r, l_r = outs[c][r]
                api.shard_scatter(o_r, len(ranks), r, out[C:C + L], plan.interleave[c], stream=streams[inst])
                if want_lse:
                    idx = _rank_lse_index(plan, c, r, device)
                    lse.index_copy_(1, idx, l_r)
    for s in streams:
        cur.wait_stream(s)
    for cm in comms:
        cm.check()
    return out, lse


def prepare_shards(q, k, v, plan: api.Plan, streams=None):
    """Per chunk, per ring rank: (q, k, v) shards under the chunk's interleave."""
    shards = []
    for c, (L, ranks) in enumerate(plan.chunks):
        C = plan.chunk_start(c)
        s = len(ranks)
        per = []
        for r in range(s):
            il = plan.interleave[c]
            per.append((api.shard_gather(q[C:C + L], s, r, il), api.shard_gather(k[C:C + L], s, r, il),
                        api.shard_gather(v[C:C + L], s, r, il)))
        shards.append(per)
    return shards


def alloc_out_shards(plan: api.Plan, Hq: int, D: int, dtype, device, want_lse=True):
    outs = []
    for L, ranks in plan.chunks:
        m2 = L // len(ranks)
        outs.append([(torch.empty((m2, Hq, D), dtype=dtype, device=device),
                      torch.empty((Hq, m2), dtype=torch.float32, device=device) if want_lse else None)
                     for _ in ranks])
    return outs


def run_plan_distributed(q_shards, k_shards, v_shards, plan: api.Plan, comm: api.Comm, softmax_scale=0.0,
                         out_shards=None, lse_shards=None, stream=None):
    """Execute, on this process's instance, every chunk whose group contains it.
    *_shards[c] = this rank's zigzag shard of chunk c (or None if not in the group)."""
    comm.reset(stream)
    outs = []
    for c, (L, ranks) in enumerate(plan.chunks):
        if comm.rank not in ranks:
            outs.append(None)
            continue
        o = out_shards[c] if out_shards is not None else torch.empty_like(q_shards[c])
        l = lse_shards[c] if lse_shards is not None else None
        api.prefill_chunk(q_shards[c], k_shards[c], v_shards[c], comm.kvstore(), api.SpGroup(comm, plan, c),
                          softmax_scale, o, l, stream=stream)
        outs.append(o)
    return outs


def run_plan_loopback_layers(qkv_layers, plan: api.Plan, comms: List[api.Comm], softmax_scale: float = 0.0,
                             streams: Optional[Sequence[torch.cuda.Stream]] = None, between=None):
    """Layer-wise CDSP prefill on loopback instances (cdsp_prefill_chunk_layer).

    qkv_layers[l] = (q, k, v) full-prompt tensors of layer l.  For every chunk, layers are
    called in order on every ring rank; ``between(layer, chunk, rank, stream)`` (optional) runs
    the caller's per-layer work (e.g. an FC stand-in) on each rank's stream after its layer call
    — the window the next layer's cache balancing overlaps (Fig. 6-b).
    Returns per layer (out [N,Hq,D], lse [Hq,N])."""
    q0 = qkv_layers[0][0]
    device = q0.device
    N, Hq, D = q0.shape
    n_layers = len(qkv_layers)
    world = len(comms)
    if streams is None:
        streams = [torch.cuda.Stream(device=device) for _ in range(world)]
    cur = torch.cuda.current_stream(device)
    for s in streams:
        s.wait_stream(cur)
    for cm in comms:
        cm.reset(cur)
    shards = [prepare_shards(q, k, v, plan) for q, k, v in qkv_layers]
    for s in streams:
        s.wait_stream(cur)
    outs = [alloc_out_shards(plan, Hq, D, q0.dtype, device) for _ in range(n_layers)]
    res = [(torch.empty_like(q0), torch.empty((Hq, N), dtype=torch.float32, device=device)) for _ in range(n_layers)]
    for c, (L, ranks) in enumerate(plan.chunks):
        for l in range(n_layers):
            for r, inst in enumerate(ranks):
                qs, ks, vs = shards[l][c][r]
                o_r, l_r = outs[l][c][r]
                api.prefill_chunk(qs, ks, vs, comms[inst].kvstore(l), api.SpGroup(comms[inst], plan, c),
                                  softmax_scale, o_r, l_r, stream=streams[inst], layer=l)
            if between is not None:
                for r, inst in enumerate(ranks):
                    with torch.cuda.stream(streams[inst]):
                        between(l, c, r, streams[inst])
    C = 0
    for c, (L, ranks) in enumerate(plan.chunks):
        for r, inst in enumerate(ranks):
            idx = _rank_lse_index(plan, c, r, device)
            for l in range(n_layers):
                o_r, l_r = outs[l][c][r]
                with torch.cuda.stream(streams[inst]):
                    api.shard_scatter(o_r, len(ranks), r, res[l][0][C:C + L], plan.interleave[c], stream=streams[inst])
                    res[l][1].index_copy_(1, idx, l_r)
        C += L
    for s in streams:
        cur.wait_stream(s)
    for cm in comms:
        cm.check()
    return res
