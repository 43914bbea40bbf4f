"""External pin of the decode paged layout (R15, P:55 PagedAttention, "reuses some components
of vLLM"): the caches cdsp_kv_transfer_to_decode writes are read by an independent paged-attention
implementation — flashinfer's batch decode over an NHD paged cache ([num_pages, page_size,
kv_heads, head_dim], page table = our block table) — and its output for the newest token must equal
the oracle's attention over the ORIGINAL (unpaged) keys and values.  A wrong page order, token
order within a page or head split would scramble flashinfer's view of the cache."""
import math

import numpy as np
import pytest
import torch

import oracle
from cdsp_inputs import block_table, qkv
from paper_2511_06247_b200 import api

pytestmark = pytest.mark.gpu

flashinfer = pytest.importorskip("flashinfer")


@pytest.mark.parametrize("N,tp,B", [(4096, 8, 16), (3000, 2, 16), (2048, 1, 32)])
def test_flashinfer_reads_our_paged_layout(N, tp, B):
    Hq, Hkv, D = 32, 8, 128
    q, k, v = qkv(N, Hq, Hkv, D, torch.bfloat16, seed=N + tp)
    n_logical = (N + B - 1) // B
    num_blocks = n_logical + 24
    bt = block_table(n_logical, num_blocks, seed=3)
    kc = [torch.zeros((num_blocks, B, Hkv // tp, D), dtype=torch.bfloat16, device="cuda") for _ in range(tp)]
    vc = [torch.zeros_like(x) for x in kc]
    plan = api.Plan([(N - N % 2, [0])]) if N % 2 else api.Plan([(N, [0])])
    L = plan.chunks[0][0]
    comm = api.Comm(0, 1, 0, L, Hkv, D, torch.bfloat16)
    api.kv_transfer_to_decode(k[:L].cuda(), v[:L].cuda(), api.SpGroup(comm, plan, 0),
                              api.DecodeTarget(kc, vc, B, bt.cuda()))
    torch.cuda.synchronize()
    comm.close()
    n_ctx = L
    scale = 1.0 / math.sqrt(D)
    o_ref, _ = oracle.causal_rows(q[:L].float().numpy(), k[:L].float().numpy(), v[:L].float().numpy(), scale,
                                  rows=np.array([n_ctx - 1]))
    ws = torch.empty(128 << 20, dtype=torch.uint8, device="cuda")
    n_pages = (n_ctx + B - 1) // B
    indptr = torch.tensor([0, n_pages], dtype=torch.int32, device="cuda")
    indices = bt[:n_pages].to(torch.int32).cuda()
    last = torch.tensor([n_ctx - (n_pages - 1) * B], dtype=torch.int32, device="cuda")
    hq_t, hkv_t = Hq // tp, Hkv // tp
    for t in range(tp):
        w = flashinfer.BatchDecodeWithPagedKVCacheWrapper(ws, "NHD")
        w.plan(indptr, indices, last, hq_t, hkv_t, D, B, q_data_type=torch.bfloat16, kv_data_type=torch.bfloat16)
        qt = q[n_ctx - 1:n_ctx, t * hq_t:(t + 1) * hq_t].contiguous().cuda()
        o = w.run(qt, (kc[t], vc[t]))
        torch.cuda.synchronize()
        err = np.abs(o.float().cpu().numpy() - o_ref[0, t * hq_t:(t + 1) * hq_t]).max()
        assert err <= 2e-2, (t, err)
