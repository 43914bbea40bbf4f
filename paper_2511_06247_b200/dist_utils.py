"""Host-side plumbing for one-process-per-GPU runs (torch.distributed): IPC-handle exchange,
plan consistency across ranks, max-over-ranks timing.  No data-path work happens here —
the ring moves KV with the library's copy-engine pulls over NVLink."""
from __future__ import annotations

import hashlib
from typing import List, Sequence

import torch
import torch.distributed as dist


def exchange_bytes(blob: bytes, group=None) -> List[bytes]:
    """All-gather one small byte string per rank (e.g. a 64-byte cudaIpcMemHandle)."""
    out = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, bytes(blob), group=group)
    return [bytes(x) for x in out]


def plan_digest(chunks: Sequence[tuple]) -> str:
    """Stable digest of a CDSP plan [(len, ring-order ranks)]; collective calls need every
    rank of a chunk's group to pass the identical plan (cdsp.h, NCCL-like semantics)."""
    h = hashlib.sha256()
    for L, ranks in chunks:
        h.update(f"{int(L)}:{','.join(str(int(r)) for r in ranks)};".encode())
    return h.hexdigest()


def check_plan_consistent(chunks: Sequence[tuple], group=None) -> None:
    digests = exchange_bytes(plan_digest(chunks).encode(), group)
    if len(set(digests)) != 1:
        raise RuntimeError(f"ranks disagree on the CDSP plan: {sorted(set(d.decode()[:12] for d in digests))}")


def max_over_ranks(values: Sequence[float], group=None, device=None) -> List[float]:
    """Element-wise max over ranks (timings are reported as the slowest rank)."""
    t = torch.tensor(list(values), dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return t.tolist()
