"""GPU parity of the whole CDSP path (cdsp_prefill_chunk, loopback ring on one B200) and of
the decode KV transfer, against the CPU oracle.

Invariants (north_star): the ring, SP-sharded result equals single-device attention; the
output is invariant to the chunking plan and per-chunk SP sizes (each plan is checked
against the oracle, R19); the balanced store layout and the paged KV layout are bit-exact."""
import math

import numpy as np
import pytest
import torch

import oracle
from tolerances import assert_out_close
from cdsp_inputs import block_table, qkv, sample_rows
from paper_2511_06247_b200 import api
from paper_2511_06247_b200.driver import make_loopback_comms, run_plan_loopback

pytestmark = pytest.mark.gpu

TOL = {torch.bfloat16: 2e-2, torch.float32: 1e-4}
LSE_TOL = 1e-3


def _run_and_check(plan_list, N, Hq, Hkv, D, dtype, rows=None, seed=0, sharp=False):
    q, k, v = qkv(N, Hq, Hkv, D, dtype, seed=seed, sharp=sharp)
    plan = api.Plan(plan_list)
    comms = make_loopback_comms(plan, Hkv, D, dtype, Hq=Hq)
    out, lse = run_plan_loopback(q.cuda(), k.cuda(), v.cuda(), plan, comms=comms)
    torch.cuda.synchronize()
    scale = 1.0 / math.sqrt(D)
    o_ref, l_ref = oracle.causal_rows(q.float().numpy(), k.float().numpy(), v.float().numpy(), scale, rows=rows)
    o = out.float().cpu().numpy()
    l = lse.cpu().numpy()
    if rows is not None:
        o, l = o[rows], l[:, rows]
    err = np.abs(o - o_ref).max()
    lerr = np.abs(l - l_ref).max()
    assert_out_close(o, o_ref, dtype == torch.bfloat16, str(plan_list))
    assert lerr <= LSE_TOL, f"{plan_list}: lse max-abs {lerr:.3e}"
    return comms, (q, k, v), plan


# M1 (BASELINE configs[0]): 1 request, 1K tokens, SP=2, 4 heads, d=64, fp32 — every row.
M1_PLANS = [
    [(1024, [0, 1])],
    [(512, [0]), (512, [0, 1])],
    [(256, [0, 1]), (256, [0, 1]), (512, [0, 1])],
    [(1024, [0])],
]


@pytest.mark.parametrize("plan", M1_PLANS)
def test_m1_tiny_fp32_all_rows(plan):
    comms, _, _ = _run_and_check(plan, 1024, 4, 4, 64, torch.float32)
    for c in comms:
        c.close()


BF16_PLANS = [
    ([(2048, [0, 1])], 2048),
    ([(2048, [0, 1, 2, 3])], 2048),
    ([(4096, list(range(8)))], 4096),
    ([(512, [0, 1]), (512, [0, 1, 2, 3]), (1024, list(range(8))), (1024, list(range(8)))], 3072),
    ([(768, [0, 1]), (1536, [0, 1, 2, 3]), (2560, list(range(8)))], 4864),
    ([(1000, [2]), (1000, [2, 5]), (2000, [2, 5, 0, 7])], 4000),
]


@pytest.mark.parametrize("plan,N", BF16_PLANS)
@pytest.mark.parametrize("heads", [(4, 4), (8, 2)])
def test_ring_bf16_matches_oracle(plan, N, heads):
    Hq, Hkv = heads
    comms, _, _ = _run_and_check(plan, N, Hq, Hkv, 128, torch.bfloat16, seed=len(plan))
    for c in comms:
        c.close()


def test_ring_sharp_queries():
    comms, _, _ = _run_and_check([(2048, [0, 1]), (2048, [0, 1, 2, 3])], 4096, 4, 2, 128, torch.bfloat16,
                                 sharp=True, seed=9)
    for c in comms:
        c.close()


def test_balanced_store_layout_bit_exact():
    """After every chunk, each instance's store holds exactly the oracle's positions (R8), in
    order, and the K/V rows of those positions, bit for bit."""
    plan_list = [(512, [0, 1]), (512, [0, 1, 2, 3]), (1024, list(range(8)))]
    N, Hq, Hkv, D = 2048, 4, 2, 128
    comms, (q, k, v), plan = _run_and_check(plan_list, N, Hq, Hkv, D, torch.bfloat16, seed=4)
    last_L, last_ranks = plan_list[-1]
    ext = plan_list + [(2 * len(last_ranks), last_ranks)]
    n, pos, _ = oracle.plan_stores(ext, len(plan_list))
    for i, inst in enumerate(last_ranks):
        st = comms[inst].kvstore()
        assert st.n == n[i]
        got_pos = st.pos[: st.n].cpu().numpy().astype(np.int64)
        np.testing.assert_array_equal(got_pos, pos[i])
        assert torch.equal(st.k[: st.n].cpu(), k[torch.as_tensor(pos[i])])
        assert torch.equal(st.v[: st.n].cpu(), v[torch.as_tensor(pos[i])])
    for c in comms:
        c.close()


def test_plan_invariance_three_plans_same_prompt():
    """Plans A, B and a single chunk over the same prompt each match the oracle."""
    N = 4096
    for plan in ([(1024, [0, 1]), (1024, [0, 1, 2, 3]), (2048, list(range(8)))],
                 [(512, [0, 1]), (1536, [0, 1, 2, 3]), (2048, list(range(8)))],
                 [(4096, list(range(8)))]):
        rows = sample_rows(N, 256, seed=2, edges=[0, 511, 512, 1023, 1024, 2047, 2048, 4095]).numpy()
        comms, _, _ = _run_and_check(plan, N, 8, 2, 128, torch.bfloat16, rows=rows, seed=21)
        for c in comms:
            c.close()


def test_m2_shape_sp8_sampled():
    """BASELINE configs[1]: 7B-shaped MHA 32K, single chunk, SP=8 ring (loopback)."""
    N = 32768
    rows = sample_rows(N, 40, seed=3, edges=[0, 2047, 2048, 4095, 4096, 30719, 30720, N - 1]).numpy()
    comms, _, _ = _run_and_check([(N, list(range(8)))], N, 32, 32, 128, torch.bfloat16, rows=rows, seed=0)
    for c in comms:
        c.close()


def test_prefill_rejects_bad_calls():
    plan = api.Plan([(256, [0, 1])])
    comms = make_loopback_comms(plan, 2, 128, torch.bfloat16)
    q = torch.zeros(128, 4, 128, dtype=torch.bfloat16, device="cuda")
    kv = torch.zeros(128, 2, 128, dtype=torch.bfloat16, device="cuda")
    g = api.SpGroup(comms[0], plan, 0)
    with pytest.raises(api.CdspError) as e:  # wrong shard length
        api.prefill_chunk(q[:64], kv[:64], kv[:64], comms[0].kvstore(), g)
    assert e.value.status == 2
    with pytest.raises(api.CdspError) as e:  # dtype mismatch
        api.prefill_chunk(q.float(), kv, kv, comms[0].kvstore(), g)
    assert e.value.status == 3
    with pytest.raises(api.CdspError) as e:  # instance not in the group
        other = api.Comm(0, 3, 0, 256, 2, 128)
        api.prefill_chunk(q, kv, kv, other.kvstore(), api.SpGroup(other, api.Plan([(256, [1, 2])]), 0))
    assert e.value.status == 4
    with pytest.raises(api.CdspError) as e:  # store of another communicator
        api.prefill_chunk(q, kv, kv, comms[1].kvstore(), g)
    assert e.value.status == 1
    for c in comms:
        c.close()


@pytest.mark.parametrize("tp", [8, 2, 1])
def test_kv_transfer_to_decode_bit_exact(tp):
    """M4 shape in miniature: GQA 32/8, plan [L@2, L@4, 2L@8]; the ENTIRE paged K/V caches
    equal the oracle writer's (sentinel-filled untouched blocks included)."""
    Hkv, D, B = 8, 128, 16
    plan_list = [(512, [0, 1]), (512, [0, 1, 2, 3]), (1024, list(range(8)))]
    N = 2048
    _, k, v = qkv(N, 32, Hkv, D, torch.bfloat16, seed=5)
    plan = api.Plan(plan_list)
    n_logical = N // B
    num_blocks = n_logical + 40
    bt = block_table(n_logical, num_blocks, seed=7)
    # sentinel 0x7FBF (a NaN bit pattern no bf16 input holds) in every untouched slot
    kc = [torch.full((num_blocks, B, Hkv // tp, D), 0x7FBF, dtype=torch.int16, device="cuda").view(torch.bfloat16)
          for _ in range(tp)]
    vc = [t.clone() for t in kc]
    dst = api.DecodeTarget(kc, vc, B, bt.cuda())
    comm = make_loopback_comms(plan, Hkv, D, torch.bfloat16)
    kd, vd = k.cuda(), v.cuda()
    for c, (L, ranks) in enumerate(plan_list):
        C = plan.chunk_start(c)
        for r, inst in enumerate(ranks):
            ks = api.zigzag_gather(kd[C:C + L], len(ranks), r)
            vs = api.zigzag_gather(vd[C:C + L], len(ranks), r)
            api.kv_transfer_to_decode(ks, vs, api.SpGroup(comm[inst], plan, c), dst)
            assert api.kv_transfer_errors(comm[inst]) == 0
    torch.cuda.synchronize()
    ok = [np.full((num_blocks, B, Hkv // tp, D), 0x7FBF, np.uint16) for _ in range(tp)]
    ov = [x.copy() for x in ok]
    kb = k.view(torch.int16).numpy().view(np.uint16)
    vb = v.view(torch.int16).numpy().view(np.uint16)
    oracle.paged_write(kb, np.arange(N), tp, B, bt.numpy(), ok)
    oracle.paged_write(vb, np.arange(N), tp, B, bt.numpy(), ov)
    for t in range(tp):
        assert np.array_equal(kc[t].cpu().view(torch.int16).numpy().view(np.uint16), ok[t])
        assert np.array_equal(vc[t].cpu().view(torch.int16).numpy().view(np.uint16), ov[t])
    for c in comm:
        c.close()


def test_kv_transfer_rejects_tp_above_hkv():
    plan = api.Plan([(256, [0])])
    comm = api.Comm(0, 1, 0, 256, 2, 128)
    k = torch.zeros(256, 2, 128, dtype=torch.bfloat16, device="cuda")
    caches = [torch.zeros(32, 16, 1, 128, dtype=torch.bfloat16, device="cuda") for _ in range(4)]
    dst = api.DecodeTarget(caches, caches, 16, torch.arange(16, dtype=torch.int32, device="cuda"))
    with pytest.raises(api.CdspError) as e:
        api.kv_transfer_to_decode(k, k, api.SpGroup(comm, plan, 0), dst)
    assert e.value.status == 8
    comm.close()


def test_kv_transfer_counts_bad_block_ids():
    plan = api.Plan([(64, [0])])
    comm = api.Comm(0, 1, 0, 64, 1, 64, torch.bfloat16)
    k = torch.ones(64, 1, 64, dtype=torch.bfloat16, device="cuda")
    caches = [torch.zeros(4, 16, 1, 64, dtype=torch.bfloat16, device="cuda")]
    bt = torch.tensor([0, 1, 99, 3], dtype=torch.int32, device="cuda")  # block 2 -> 99 out of range
    api.kv_transfer_to_decode(k, k, api.SpGroup(comm, plan, 0), api.DecodeTarget(caches, caches, 16, bt))
    assert api.kv_transfer_errors(comm) == 16
    comm.close()
