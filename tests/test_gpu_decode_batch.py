"""GPU parity of the batched decode step (cdsp_decode_attention_batch): every request's newest
token over its own pages of one shared paged pool must equal the oracle's attention over that
request's unpaged k/v (R1, R2, R4, R14, R15).

Each request's cache rows are written through the product's transfer call (layout pinned
bit-exactly against the oracle writer elsewhere) into a disjoint, seeded slice of the pool;
rows no request owns hold NaN, table entries past a request's pages are -1."""
import math

import numpy as np
import pytest
import torch

import oracle
from cdsp_inputs import qkv
from paper_2511_06247_b200 import api

pytestmark = pytest.mark.gpu

TOL, LSE_TOL = 2e-2, 1e-3


def _batch(lens, Hq, Hkv, D, tp, B=16, seed=3):
    """Per request: (q, k, v) with k/v of lens[b] tokens (even length for the s=1 transfer plan),
    written into one pool through row b of a [batch, pages] block table."""
    g = torch.Generator().manual_seed(seed)
    pages = [(n + B - 1) // B for n in lens]
    row = max(pages)
    pool = sum(pages) + 16
    perm = torch.randperm(pool, generator=g).to(torch.int32)
    bt = torch.full((len(lens), row), -1, dtype=torch.int32)
    o = 0
    for b, n in enumerate(pages):
        bt[b, :n] = perm[o:o + n]
        o += n
    bt = bt.cuda()
    kc = [torch.full((pool, B, Hkv // tp, D), float("nan"), dtype=torch.bfloat16, device="cuda") for _ in range(tp)]
    vc = [torch.full_like(x, float("nan")) for x in kc]
    reqs = []
    for b, n in enumerate(lens):
        N = n + (n % 2)
        q, k, v = qkv(N, Hq, Hkv, D, torch.bfloat16, seed=seed * 100 + b)
        dst_b = api.DecodeTarget(kc, vc, B, bt[b])  # row b (contiguous) as a one-request table
        comm = api.Comm(0, 1, 0, N, Hkv, D, torch.bfloat16)
        api.kv_transfer_to_decode(k.cuda(), v.cuda(), api.SpGroup(comm, api.Plan([(N, [0])]), 0), dst_b)
        assert api.kv_transfer_errors(comm) == 0
        comm.close()
        reqs.append((q[n - 1:n], k, v))
    return api.DecodeTarget(kc, vc, B, bt), reqs


def _check(lens, Hq, Hkv, D, tp, ranks, B=16):
    dst, reqs = _batch(lens, Hq, Hkv, D, tp, B)
    hq_t, hkv_t = Hq // tp, Hkv // tp
    for t in ranks:
        q = torch.cat([r[0][:, t * hq_t:(t + 1) * hq_t] for r in reqs]).contiguous().cuda()
        lse = torch.empty((len(lens), hq_t), dtype=torch.float32, device="cuda")
        out, _ = api.decode_attention_batch(q, dst, t, hkv_t, lens, lse=lse)
        torch.cuda.synchronize()
        for b, (qb, k, v) in enumerate(reqs):
            n = lens[b]
            ks = k[:n, t * hkv_t:(t + 1) * hkv_t].float().numpy()
            vs = v[:n, t * hkv_t:(t + 1) * hkv_t].float().numpy()
            o_ref, l_ref = oracle.attention(qb[:, t * hq_t:(t + 1) * hq_t].float().numpy(), np.array([n - 1]),
                                            ks, vs, np.arange(n), 1.0 / math.sqrt(D))
            err = float(np.abs(out[b:b + 1].float().cpu().numpy() - o_ref).max())
            lerr = float(np.abs(lse[b].cpu().numpy() - l_ref[:, 0]).max())
            assert err <= TOL, f"rank {t} request {b} (ctx {n}): out max-abs {err:.3e}"
            assert lerr <= LSE_TOL, f"rank {t} request {b} (ctx {n}): lse max-abs {lerr:.3e}"


@pytest.mark.parametrize("heads", [(32, 8, 8), (16, 8, 2), (64, 8, 8)])
@pytest.mark.parametrize("D", [128, 64])
def test_batch_mixed_lengths(heads, D):
    Hq, Hkv, tp = heads
    _check([1000, 17, 5003, 1, 4096], Hq, Hkv, D, tp, sorted({0, tp - 1}))


def test_batch_equal_lengths_many_requests():
    _check([2048] * 12, 32, 8, 128, 8, [0, 3])


def test_batch_many_short_and_one_long():
    """300 requests of 16..700 tokens and one of 20000: the split search and the 1D grid's
    binary search over 301 request offsets."""
    g = torch.Generator().manual_seed(9)
    lens = [int(x) for x in torch.randint(16, 701, (300,), generator=g)] + [20000]
    _check(lens, 32, 8, 128, 8, [0])


def test_batch_of_one_equals_single_call():
    """batch = 1 through the batch entry point == cdsp_decode_attention (same kernel, same splits)."""
    dst, reqs = _batch([3001], 32, 8, 128, 8)
    q = reqs[0][0][:, :4].contiguous().cuda()
    ob, _ = api.decode_attention_batch(q, dst, 0, 1, [3001])
    single = api.DecodeTarget(dst.k_caches, dst.v_caches, 16, dst.block_table[0])
    os_, _ = api.decode_attention(q, single, 0, 1, 3001)
    torch.cuda.synchronize()
    assert torch.equal(ob, os_)


def test_batch_refusals():
    dst, reqs = _batch([64, 64], 32, 8, 128, 8)
    q = torch.zeros((2, 4, 128), dtype=torch.bfloat16, device="cuda")
    with pytest.raises(api.CdspError, match="SHAPE"):  # out rows != batch
        api.decode_attention_batch(q, dst, 0, 1, [64, 64], out=torch.empty_like(q[:1]))
    with pytest.raises(api.CdspError, match="SHAPE"):  # an empty request
        api.decode_attention_batch(q, dst, 0, 1, [64, 0])
    with pytest.raises(api.CdspError, match="CAPACITY"):  # a table row covers 64 positions
        api.decode_attention_batch(q, dst, 0, 1, [64, 65])
    small = api.DecodeTarget([x.view(-1, 8, 1, 128) for x in dst.k_caches],
                             [x.view(-1, 8, 1, 128) for x in dst.v_caches], 8, dst.block_table)
    with pytest.raises(api.CdspError, match="UNSUPPORTED"):  # block 8: not the TMA kernel
        api.decode_attention_batch(q, small, 0, 1, [16, 16])


def test_batch_bench_shape_32x32k():
    """The bench's launch configuration (tools/bench_decode_batch.py, 32 requests x 32K on a rank
    with 4 query heads / 1 KV head: 32 virtual heads x 9 splits, one wave): sampled requests vs
    the oracle."""
    lens = [32768] * 32
    dst, reqs = _batch(lens, 4, 1, 128, 1)
    q = torch.cat([r[0] for r in reqs]).contiguous().cuda()
    lse = torch.empty((32, 4), dtype=torch.float32, device="cuda")
    out, _ = api.decode_attention_batch(q, dst, 0, 1, lens, lse=lse)
    torch.cuda.synchronize()
    for b in (0, 13, 31):
        qb, k, v = reqs[b]
        o_ref, l_ref = oracle.attention(qb.float().numpy(), np.array([32767]), k.float().numpy(), v.float().numpy(),
                                        np.arange(32768), 1.0 / math.sqrt(128))
        assert float(np.abs(out[b:b + 1].float().cpu().numpy() - o_ref).max()) <= TOL, b
        assert float(np.abs(lse[b].cpu().numpy() - l_ref[:, 0]).max()) <= LSE_TOL, b
