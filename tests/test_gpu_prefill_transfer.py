"""cdsp_prefill_chunk_transfer (rows a4 + a7 in one call): the chunk's attention and its KV
transfer into the decode caches (R15), the scatter on the communicator's transfer
stream overlapping the attention.  The result must be exactly what the two separate calls on one
stream produce:
  * the ENTIRE paged caches equal the oracle writer's (sentinel in every untouched slot);
  * out / lse are bit-identical to cdsp_prefill_chunk's (and match the oracle);
  * block-table entries out of range are skipped and counted like the scatter kernel counts;
  * a chunk with history and the caller's stream ordering (results read on that stream)."""
import math

import numpy as np
import pytest
import torch

import oracle
from tolerances import assert_out_close
from cdsp_inputs import block_table, qkv, sample_rows
from paper_2511_06247_b200 import api

pytestmark = pytest.mark.gpu

SENT = 0x7FBF  # a NaN bit pattern no bf16 input holds


def _caches(num_blocks, B, hkv_t, D, tp):
    kc = [torch.full((num_blocks, B, hkv_t, D), SENT, dtype=torch.int16, device="cuda").view(torch.bfloat16)
          for _ in range(tp)]
    return kc, [t.clone() for t in kc]


def _u16(t):
    return t.cpu().view(torch.int16).numpy().view(np.uint16)


def _expect(k, v, pos, tp, B, bt, num_blocks, hkv_t, D):
    ok = [np.full((num_blocks, B, hkv_t, D), SENT, np.uint16) for _ in range(tp)]
    ov = [x.copy() for x in ok]
    oracle.paged_write(_u16(k), pos, tp, B, bt, ok)
    oracle.paged_write(_u16(v), pos, tp, B, bt, ov)
    return ok, ov


@pytest.mark.parametrize("L,Hq,Hkv,tp,B", [
    (4096, 8, 8, 8, 16),     # MHA, one KV head per decode rank
    (4096, 32, 8, 8, 16),    # GQA 4: only the first query head of each group writes
    (3072, 16, 4, 2, 32),    # two heads per decode rank, 32-token pages
    (2048, 8, 2, 1, 64),     # one decode rank holding every head, 64-token pages
    (1040, 4, 4, 4, 16),     # chunk not a multiple of the 256-row pair: a lone last row block
    (4096, 8, 8, 8, 8),      # 8-token pages
    (1000, 8, 8, 8, 16),     # a ragged last page
])
def test_prefill_transfer_equals_separate_calls(L, Hq, Hkv, tp, B):
    D = 128
    q, k, v = qkv(L, Hq, Hkv, D, torch.bfloat16, seed=L + Hq + B)
    qd, kd, vd = q.cuda(), k.cuda(), v.cuda()
    plan = api.Plan([(L, [0])])
    n_logical = (L + B - 1) // B
    num_blocks = n_logical + 24
    bt = block_table(n_logical, num_blocks, seed=B)
    hkv_t = Hkv // tp
    results = {}
    for fused in (True, False):
        comm = api.Comm(0, 1, 0, L, Hkv, D, torch.bfloat16)
        kc, vc = _caches(num_blocks, B, hkv_t, D, tp)
        dst = api.DecodeTarget(kc, vc, B, bt.cuda())
        out = torch.empty_like(qd)
        lse = torch.empty(Hq, L, dtype=torch.float32, device="cuda")
        if fused:
            api.prefill_chunk_transfer(qd, kd, vd, comm.kvstore(), api.SpGroup(comm, plan, 0), dst, 0.0, out, lse)
        else:
            api.prefill_chunk(qd, kd, vd, comm.kvstore(), api.SpGroup(comm, plan, 0), 0.0, out, lse)
            api.kv_transfer_to_decode(kd, vd, api.SpGroup(comm, plan, 0), dst)
        torch.cuda.synchronize()
        assert api.kv_transfer_errors(comm) == 0
        results[fused] = (out.cpu(), lse.cpu(), [_u16(t) for t in kc], [_u16(t) for t in vc])
        comm.close()
    ok, ov = _expect(k, v, np.arange(L), tp, B, bt.numpy(), num_blocks, hkv_t, D)
    for t in range(tp):
        assert np.array_equal(results[True][2][t], ok[t]), f"K cache of decode rank {t}"
        assert np.array_equal(results[True][3][t], ov[t]), f"V cache of decode rank {t}"
        assert np.array_equal(results[False][2][t], ok[t]) and np.array_equal(results[False][3][t], ov[t])
    assert torch.equal(results[True][0], results[False][0]), "attention output differs from cdsp_prefill_chunk"
    assert torch.equal(results[True][1], results[False][1]), "lse differs from cdsp_prefill_chunk"
    rows = sample_rows(L, 64, seed=3, edges=[0, L - 1]).numpy()
    o_ref, l_ref = oracle.causal_rows(q.float().numpy(), k.float().numpy(), v.float().numpy(), 1.0 / math.sqrt(D),
                                      rows=rows)
    assert_out_close(results[True][0].float().numpy()[rows], o_ref, True, f"L={L}")
    assert np.abs(results[True][1].numpy()[:, rows] - l_ref).max() <= 1e-3


def test_prefill_transfer_counts_bad_block_ids_like_the_scatter():
    """Pages whose block-table entry is out of range are skipped (their slots keep the
    sentinel) and counted once per token, exactly as cdsp_kv_transfer_to_decode does."""
    L, Hq, Hkv, D, tp, B = 2048, 8, 8, 128, 8, 16
    q, k, v = qkv(L, Hq, Hkv, D, torch.bfloat16, seed=9)
    qd, kd, vd = q.cuda(), k.cuda(), v.cuda()
    plan = api.Plan([(L, [0])])
    n_logical = L // B
    num_blocks = n_logical + 8
    bt = block_table(n_logical, num_blocks, seed=4)
    bt[5] = -1
    bt[77] = num_blocks + 3
    bad = {}
    caches = {}
    for fused in (True, False):
        comm = api.Comm(0, 1, 0, L, Hkv, D, torch.bfloat16)
        kc, vc = _caches(num_blocks, B, Hkv // tp, D, tp)
        dst = api.DecodeTarget(kc, vc, B, bt.cuda())
        if fused:
            api.prefill_chunk_transfer(qd, kd, vd, comm.kvstore(), api.SpGroup(comm, plan, 0), dst)
        else:
            api.prefill_chunk(qd, kd, vd, comm.kvstore(), api.SpGroup(comm, plan, 0))
            api.kv_transfer_to_decode(kd, vd, api.SpGroup(comm, plan, 0), dst)
        torch.cuda.synchronize()
        bad[fused] = api.kv_transfer_errors(comm)
        caches[fused] = ([_u16(t) for t in kc], [_u16(t) for t in vc])
        comm.close()
    assert bad[True] == bad[False] == 2 * B
    for t in range(tp):
        assert np.array_equal(caches[True][0][t], caches[False][0][t])
        assert np.array_equal(caches[True][1][t], caches[False][1][t])


def test_prefill_transfer_two_chunks_with_history():
    """Two chunks (the second with history): both chunks' KV land in the caches exactly as the
    oracle writes them, and the outputs match the oracle."""
    L, Hq, Hkv, D, tp, B = 2048, 8, 8, 128, 8, 16
    q, k, v = qkv(2 * L, Hq, Hkv, D, torch.bfloat16, seed=12)
    qd, kd, vd = q.cuda(), k.cuda(), v.cuda()
    plan = api.Plan([(L, [0]), (L, [0])])
    n_logical = 2 * L // B
    num_blocks = n_logical + 8
    bt = block_table(n_logical, num_blocks, seed=6)
    comm = api.Comm(0, 1, 0, 2 * L, Hkv, D, torch.bfloat16)
    kc, vc = _caches(num_blocks, B, Hkv // tp, D, tp)
    dst = api.DecodeTarget(kc, vc, B, bt.cuda())
    out = torch.empty_like(qd)
    for c in range(2):
        sl = slice(c * L, (c + 1) * L)
        out[sl] = api.prefill_chunk_transfer(qd[sl].contiguous(), kd[sl].contiguous(), vd[sl].contiguous(),
                                             comm.kvstore(), api.SpGroup(comm, plan, c), dst)
    torch.cuda.synchronize()
    assert api.kv_transfer_errors(comm) == 0
    ok, ov = _expect(k, v, np.arange(2 * L), tp, B, bt.numpy(), num_blocks, Hkv // tp, D)
    for t in range(tp):
        assert np.array_equal(_u16(kc[t]), ok[t]) and np.array_equal(_u16(vc[t]), ov[t])
    rows = sample_rows(2 * L, 48, seed=2, edges=[0, L - 1, L, 2 * L - 1]).numpy()
    o_ref, _ = oracle.causal_rows(q.float().numpy(), k.float().numpy(), v.float().numpy(), 1.0 / math.sqrt(D),
                                  rows=rows)
    assert_out_close(out.float().cpu().numpy()[rows], o_ref, True, "two chunks")
    comm.close()


def test_prefill_transfer_loopback_ring():
    """SP = 2 then SP = 4 chunks on loopback instances: every rank's call transfers its zigzag
    shard (the group executes on the last rank's call; each rank's scatter only reads its own
    k / v): the caches equal the oracle writer's over the whole prompt, the outputs the oracle's."""
    from paper_2511_06247_b200.driver import make_loopback_comms
    Hq, Hkv, D, tp, B = 8, 4, 128, 4, 16
    plan_list = [(1024, [0, 1]), (2048, [0, 1, 2, 3])]
    N = sum(L for L, _ in plan_list)
    q, k, v = qkv(N, Hq, Hkv, D, torch.bfloat16, seed=21)
    qd, kd, vd = q.cuda(), k.cuda(), v.cuda()
    plan = api.Plan(plan_list)
    comms = make_loopback_comms(plan, Hkv, D, torch.bfloat16, Hq=Hq)
    n_logical = N // B
    num_blocks = n_logical + 8
    bt = block_table(n_logical, num_blocks, seed=8)
    kc, vc = _caches(num_blocks, B, Hkv // tp, D, tp)
    dst = api.DecodeTarget(kc, vc, B, bt.cuda())
    out = torch.empty_like(qd)
    for c, (L, ranks) in enumerate(plan_list):
        C = plan.chunk_start(c)
        s = len(ranks)
        res = []
        for r, inst in enumerate(ranks):
            qs, ks, vs = (api.zigzag_gather(t[C:C + L].contiguous(), s, r) for t in (qd, kd, vd))
            o = torch.empty_like(qs)
            api.prefill_chunk_transfer(qs, ks, vs, comms[inst].kvstore(), api.SpGroup(comms[inst], plan, c), dst,
                                       0.0, o)
            res.append((qs, ks, vs, o))
        torch.cuda.synchronize()
        part = torch.empty(L, Hq, D, dtype=torch.bfloat16, device="cuda")
        for r in range(s):
            api.zigzag_scatter(res[r][3], s, r, part)
        out[C:C + L] = part
        for inst in ranks:
            assert api.kv_transfer_errors(comms[inst]) == 0
    torch.cuda.synchronize()
    ok, ov = _expect(k, v, np.arange(N), tp, B, bt.numpy(), num_blocks, Hkv // tp, D)
    for t in range(tp):
        assert np.array_equal(_u16(kc[t]), ok[t]) and np.array_equal(_u16(vc[t]), ov[t])
    rows = sample_rows(N, 64, seed=4, edges=[0, 1023, 1024, N - 1]).numpy()
    o_ref, _ = oracle.causal_rows(q.float().numpy(), k.float().numpy(), v.float().numpy(), 1.0 / math.sqrt(D),
                                  rows=rows)
    assert_out_close(out.float().cpu().numpy()[rows], o_ref, True, str(plan_list))
    for cm in comms:
        cm.close()


def test_prefill_transfer_refuses_bad_target_before_any_work():
    """A decode target the transfer refuses (Hkv not divisible by tp) fails the call before
    anything is enqueued: the output keeps its sentinel and the store stays empty."""
    L, Hq, Hkv, D = 512, 4, 4, 128
    q, k, v = (t.cuda() for t in qkv(L, Hq, Hkv, D, torch.bfloat16, seed=2))
    plan = api.Plan([(L, [0])])
    comm = api.Comm(0, 1, 0, L, Hkv, D, torch.bfloat16)
    caches = [torch.zeros(40, 16, 1, D, dtype=torch.bfloat16, device="cuda") for _ in range(3)]
    dst = api.DecodeTarget(caches, caches, 16, torch.arange(40, dtype=torch.int32, device="cuda"))
    out = torch.full_like(q, 7.0)
    with pytest.raises(api.CdspError) as e:
        api.prefill_chunk_transfer(q, k, v, comm.kvstore(), api.SpGroup(comm, plan, 0), dst, 0.0, out)
    assert e.value.status == 8
    torch.cuda.synchronize()
    assert bool((out == 7.0).all())
    # the store was not appended: the same chunk can still be prefilled
    api.prefill_chunk(q, k, v, comm.kvstore(), api.SpGroup(comm, plan, 0), 0.0, out)
    torch.cuda.synchronize()
    comm.close()
