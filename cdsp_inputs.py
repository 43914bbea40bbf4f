"""Seeded synthetic inputs shared by the oracle side and the CUDA side of every test and
of bench.py.  This module holds NONE of the method's arithmetic: it only draws random
numbers and names workload shapes (DESIGN.md §"Input recipe").

Recipe: q, k, v are i.i.d. N(0, 1) drawn in float32 from
``torch.Generator`` seeds q=1001, k=1002, v=1003 (offset by ``seed``), then RNE-rounded to
the compute dtype.  The oracle consumes the rounded values widened to float64, so input
quantisation is not counted as error.  ``sharp=True`` scales q by 4 (stresses the
online-softmax range).  Shapes follow the paper's workloads: LLaMA3-8B-like GQA (32 Q /
8 KV heads, d=128) and a 7B-shaped MHA (32/32, d=128); prompts 1K .. 512K.
"""
from __future__ import annotations

import torch

SEED_Q, SEED_K, SEED_V = 1001, 1002, 1003


def _randn(shape, seed: int, device="cpu") -> torch.Tensor:
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    return torch.randn(*shape, generator=g, dtype=torch.float32, device=device)


def qkv(N: int, Hq: int, Hkv: int, D: int, dtype=torch.bfloat16, seed: int = 0,
        sharp: bool = False, device="cpu"):
    """Full-prompt q [N,Hq,D], k, v [N,Hkv,D] in `dtype` (drawn in fp32, RNE-rounded)."""
    q = _randn((N, Hq, D), SEED_Q + seed, device)
    if sharp:
        q = q * 4.0
    k = _randn((N, Hkv, D), SEED_K + seed, device)
    v = _randn((N, Hkv, D), SEED_V + seed, device)
    return q.to(dtype), k.to(dtype), v.to(dtype)


def block_table(n_logical: int, n_physical: int, seed: int = 7) -> torch.Tensor:
    """int32 [n_logical] distinct physical block ids drawn from [0, n_physical)."""
    g = torch.Generator()
    g.manual_seed(seed)
    return torch.randperm(n_physical, generator=g)[:n_logical].to(torch.int32)


def sample_rows(N: int, n: int, seed: int = 11, edges=()) -> torch.Tensor:
    """Sorted distinct int64 query positions: `edges` (shard / tile boundaries) plus
    uniformly drawn positions, n in total (or N if smaller)."""
    g = torch.Generator()
    g.manual_seed(seed)
    fixed = sorted({int(e) for e in edges if 0 <= int(e) < N})
    want = max(0, min(n, N) - len(fixed))
    perm = torch.randperm(N, generator=g)
    extra = [int(x) for x in perm[: want + len(fixed)].tolist() if int(x) not in set(fixed)][:want]
    return torch.tensor(sorted(set(fixed) | set(extra)), dtype=torch.int64)


# ---- named workloads (BASELINE.json configs) --------------------
# plan = list of (chunk length, ring-order instance ids)
WORKLOADS = {
    "M1_tiny": dict(N=1024, Hq=4, Hkv=4, D=64, dtype=torch.float32,
                    plan=[(1024, [0, 1])]),
    "M2_7b_mha_32k": dict(N=32768, Hq=32, Hkv=32, D=128, dtype=torch.bfloat16,
                          plan=[(32768, list(range(8)))]),
    "M3_128k_4chunk": dict(N=131072, Hq=32, Hkv=32, D=128, dtype=torch.bfloat16,
                           plan=[(32768, [0, 1]), (32768, [0, 1, 2, 3]),
                                 (32768, list(range(8))), (32768, list(range(8)))]),
    "M4_llama3_8b_256k": dict(N=262144, Hq=32, Hkv=8, D=128, dtype=torch.bfloat16,
                              plan=[(65536, [0, 1]), (65536, [0, 1, 2, 3]), (131072, list(range(8)))]),
    "M5_512k_weak": dict(N=524288, Hq=32, Hkv=8, D=128, dtype=torch.bfloat16,
                         plan=[(524288, list(range(8)))]),
}
