"""GPU parity of the decode consumer: cdsp_decode_attention reads the
paged caches written by cdsp_kv_transfer_to_decode and must equal the oracle's attention of
the newest token over every cached position (R1, R2, R4, R14, R15).

The cache is filled through the product's own transfer call (whose layout is pinned
bit-exactly against the oracle writer in test_gpu_ring / test_gpu_fullsize); the expected
values come from oracle.attention over the original, unpaged k/v."""
import math

import numpy as np
import pytest
import torch

import oracle
from cdsp_inputs import block_table, qkv
from paper_2511_06247_b200 import api

pytestmark = pytest.mark.gpu

TOL = {torch.bfloat16: 2e-2, torch.float32: 1e-4}
LSE_TOL = 1e-3


def _caches(k, v, tp, B, seed=7, spare=8, fill=0.0):
    """Fill tp paged caches with k/v [N,Hkv,D] through cdsp_kv_transfer_to_decode (s=1 plan);
    every other cache row holds `fill` (NaN: rows no token was ever written to)."""
    N, Hkv, D = k.shape
    n_logical = (N + B - 1) // B
    nb = n_logical + spare
    bt = block_table(n_logical, nb, seed=seed).cuda()
    kc = [torch.full((nb, B, Hkv // tp, D), fill, dtype=k.dtype, device="cuda") for _ in range(tp)]
    vc = [torch.full_like(x, fill) for x in kc]
    dst = api.DecodeTarget(kc, vc, B, bt)
    plan = api.Plan([(N, [0])])
    comm = api.Comm(0, 1, 0, N, Hkv, D, k.dtype)
    api.kv_transfer_to_decode(k.cuda(), v.cuda(), api.SpGroup(comm, plan, 0), dst)
    assert api.kv_transfer_errors(comm) == 0
    comm.close()
    return dst


def _check_rank(q_all, k, v, dst, t, tp, n_ctx, dtype, ws=None, kpos=None):
    Hq, Hkv, D = q_all.shape[1], k.shape[1], k.shape[2]
    hq_t, hkv_t = Hq // tp, Hkv // tp
    q_t = q_all[:, t * hq_t:(t + 1) * hq_t].contiguous()
    lse = torch.empty(hq_t, dtype=torch.float32, device="cuda")
    out, _ = api.decode_attention(q_t.cuda(), dst, t, hkv_t, n_ctx, lse=lse, workspace=ws)
    torch.cuda.synchronize()
    ks = k[:n_ctx, t * hkv_t:(t + 1) * hkv_t].float().numpy()
    vs = v[:n_ctx, t * hkv_t:(t + 1) * hkv_t].float().numpy()
    kp = np.arange(n_ctx) if kpos is None else kpos
    o_ref, l_ref = oracle.attention(q_t.float().numpy(), np.array([n_ctx - 1]), ks, vs, kp, 1.0 / math.sqrt(D))
    err = float(np.abs(out.float().cpu().numpy() - o_ref).max())
    lerr = float(np.abs(lse.cpu().numpy() - l_ref[:, 0]).max())
    assert err <= TOL[dtype], f"rank {t} n_ctx {n_ctx}: out max-abs {err:.3e}"
    assert lerr <= LSE_TOL, f"rank {t} n_ctx {n_ctx}: lse max-abs {lerr:.3e}"
    return out, lse


# (Hq, Hkv, tp) -> GQA group Hq_t / Hkv_t in {4, 1, 2, 8}
HEADS = [(32, 8, 8), (8, 8, 1), (16, 8, 2), (64, 8, 8)]


@pytest.mark.parametrize("dtype,D", [(torch.bfloat16, 128), (torch.bfloat16, 64), (torch.float32, 128),
                                     (torch.float32, 64)])
@pytest.mark.parametrize("heads", HEADS)
@pytest.mark.parametrize("n_ctx", [1, 17, 1000, 5003])
def test_decode_matches_oracle(dtype, D, heads, n_ctx):
    Hq, Hkv, tp = heads
    N = n_ctx + (n_ctx % 2)  # the s=1 transfer plan needs an even chunk length
    q, k, v = qkv(N, Hq, Hkv, D, dtype, seed=n_ctx)
    dst = _caches(k, v, tp, 16)
    qn = q[n_ctx - 1:n_ctx]  # the newest token's query
    for t in sorted({0, tp - 1}):
        _check_rank(qn, k, v, dst, t, tp, n_ctx, dtype)


@pytest.mark.parametrize("B", [1, 8, 64, 256])
def test_decode_block_sizes(B):
    n_ctx = 3000
    q, k, v = qkv(n_ctx, 32, 8, 128, torch.bfloat16, seed=B)
    dst = _caches(k, v, 8, B)
    for t in (0, 5):
        _check_rank(q[-1:], k, v, dst, t, 8, n_ctx, torch.bfloat16)


@pytest.mark.parametrize("B,n_ctx", [(16, 1000), (16, 4097), (64, 1000), (256, 3001), (8, 1000)])
def test_decode_never_written_rows_are_nan(B, n_ctx):
    """Cache rows past n_ctx in the last page (and every unused page) hold NaN, as memory no
    token was ever written to may: they must not reach the output (the TMA kernel loads whole
    16-row page pieces and zeroes V past the range; the cp.async kernel zero-fills)."""
    q, k, v = qkv(n_ctx + (n_ctx % 2), 32, 8, 128, torch.bfloat16, seed=B + n_ctx)
    dst = _caches(k, v, 8, B, fill=float("nan"))
    for t in (0, 7):
        out, lse = _check_rank(q[n_ctx - 1:n_ctx], k, v, dst, t, 8, n_ctx, torch.bfloat16)
        assert torch.isfinite(out.float()).all() and torch.isfinite(lse).all()


def test_decode_sharp_long_context_many_splits():
    """n_ctx large enough for hundreds of splits per KV head (the last-finisher slice merge
    over all of them), sharp queries (q x 4) stress the online softmax; the workspace is
    reused across calls and ranks (every call must leave its counters zeroed)."""
    n_ctx = 150001
    q, k, v = qkv(n_ctx + 1, 32, 8, 128, torch.bfloat16, seed=3, sharp=True)
    dst = _caches(k, v, 8, 16)
    ws = api.decode_workspace(4, 1, 128)
    first = None
    for t in range(8):
        out, lse = _check_rank(q[n_ctx - 1:n_ctx], k, v, dst, t, 8, n_ctx, torch.bfloat16, ws=ws)
        if t == 0:
            first = (out.clone(), lse.clone())
    out, lse = _check_rank(q[n_ctx - 1:n_ctx], k, v, dst, 0, 8, n_ctx, torch.bfloat16, ws=ws)
    assert torch.equal(out, first[0]) and torch.equal(lse, first[1]), "repeat call differs (workspace state)"
    torch.cuda.synchronize()
    assert int(ws[:512].count_nonzero()) == 0, "split counters (first 512 bytes) not reset"


def test_decode_skips_out_of_range_blocks():
    """Block-table entries outside [0, num_blocks) contribute no keys (documented behaviour)."""
    n_ctx, B = 640, 16
    q, k, v = qkv(n_ctx, 8, 2, 128, torch.bfloat16, seed=8)
    dst = _caches(k, v, 2, B)
    bt = dst.block_table
    bt[3] = -1
    bt[7] = 1 << 20
    keep = np.array([p for p in range(n_ctx) if p // B not in (3, 7)])
    Hq_t, hkv_t = 4, 1
    q_t = q[-1:, :Hq_t].contiguous()
    lse = torch.empty(Hq_t, dtype=torch.float32, device="cuda")
    out, _ = api.decode_attention(q_t.cuda(), dst, 0, hkv_t, n_ctx, lse=lse)
    torch.cuda.synchronize()
    o_ref, l_ref = oracle.attention(q_t.float().numpy(), np.array([n_ctx - 1]), k[keep, :1].float().numpy(),
                                    v[keep, :1].float().numpy(), keep, 1.0 / math.sqrt(128))
    assert np.abs(out.float().cpu().numpy() - o_ref).max() <= 2e-2
    assert np.abs(lse.cpu().numpy() - l_ref[:, 0]).max() <= 1e-3


def test_decode_rejects_bad_calls():
    q, k, v = qkv(64, 12, 4, 128, torch.bfloat16, seed=1)
    dst = _caches(k, v, 1, 16)
    qn = q[-1:].cuda()
    with pytest.raises(api.CdspError) as e:  # GQA group 3
        api.decode_attention(qn, dst, 0, 4, 64)
    assert e.value.status == 8
    with pytest.raises(api.CdspError) as e:  # context beyond the block table
        api.decode_attention(qn[:, :4], dst, 0, 4, 64 + 16 * 9)
    assert e.value.status == 5
    with pytest.raises(api.CdspError) as e:  # workspace too small
        api.decode_attention(qn[:, :4], dst, 0, 4, 64, workspace=torch.zeros(256, dtype=torch.uint8, device="cuda"))
    assert e.value.status == 5
    with pytest.raises(api.CdspError) as e:  # dtype mismatch q / out
        api.decode_attention(qn[:, :4], dst, 0, 4, 64, out=torch.empty(1, 4, 128, device="cuda"))
    assert e.value.status == 3
