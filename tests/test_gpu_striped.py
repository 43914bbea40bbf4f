"""GPU parity of the striped interleave ("evenly-spaced stripes ...
round-robin", "striped/zigzag"; reading R20): the same ring path with every ring step's
mask a shifted causal one (positions step by s).  Maps and layouts bit-exact, attention
within the north_star tolerances, against the CPU oracle."""
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


@pytest.mark.parametrize("s", [1, 2, 4, 8])
@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
def test_striped_gather_scatter_bit_exact(s, dtype):
    L = 2 * s * 37
    x = torch.randn(L, 3, 64, device="cuda").to(dtype)
    tr, ts = oracle.striped_map(L, s)
    full = torch.zeros_like(x)
    for r in range(s):
        sh = api.striped_gather(x, s, r)
        assert torch.equal(sh.cpu(), x.cpu()[torch.as_tensor(np.nonzero(tr == r)[0])])
        api.striped_scatter(sh, s, r, full)
    assert torch.equal(full, x)


def _check(plan_list, N, Hq, Hkv, D, dtype, rows=None, seed=0, sharp=False):
    q, k, v = qkv(N, Hq, Hkv, D, dtype, seed=seed, sharp=sharp)
    plan = api.Plan(plan_list)
    comms = make_loopback_comms(plan, Hkv, D, dtype, Hq=Hq)
    out, lse = run_plan_loopback(q.cuda(), k.cuda(), v.cuda(), plan, comms=comms)
    torch.cuda.synchronize()
    o_ref, l_ref = oracle.causal_rows(q.float().numpy(), k.float().numpy(), v.float().numpy(),
                                      1.0 / math.sqrt(D), rows=rows)
    o, l = out.float().cpu().numpy(), lse.cpu().numpy()
    if rows is not None:
        o, l = o[rows], l[:, rows]
    assert_out_close(o, o_ref, dtype == torch.bfloat16, str(plan_list))
    assert np.abs(l - l_ref).max() <= 1e-3, plan_list
    return comms, (q, k, v)


PLANS = [
    ([(2048, [0, 1], "striped")], 2048),
    ([(2048, [0, 1, 2, 3], "striped")], 2048),
    ([(4096, list(range(8)), "striped")], 4096),
    ([(512, [0, 1], "striped"), (512, [0, 1, 2, 3]), (1024, list(range(8)), "striped")], 2048),
    ([(768, [0, 1]), (1536, [0, 1, 2, 3], "striped"), (2560, list(range(8)), "striped")], 4864),
    ([(1000, [2], "striped"), (1000, [2, 5], "striped"), (2000, [2, 5, 0, 7], "striped")], 4000),
]


@pytest.mark.parametrize("plan,N", PLANS)
@pytest.mark.parametrize("heads", [(4, 4), (8, 2)])
def test_striped_ring_bf16_matches_oracle(plan, N, heads):
    comms, _ = _check(plan, N, heads[0], heads[1], 128, torch.bfloat16, seed=len(plan) + 3)
    for c in comms:
        c.close()


@pytest.mark.parametrize("plan", [[(1024, [0, 1], "striped")],
                                  [(512, [0], "striped"), (512, [0, 1], "striped")],
                                  [(256, [0, 1]), (256, [0, 1], "striped"), (512, [0, 1], "striped")]])
def test_striped_m1_fp32_all_rows(plan):
    comms, _ = _check(plan, 1024, 4, 4, 64, torch.float32)
    for c in comms:
        c.close()


def test_striped_sharp_and_m2_shape_sampled():
    comms, _ = _check([(2048, [0, 1], "striped"), (2048, [0, 1, 2, 3], "striped")], 4096, 4, 2, 128,
                      torch.bfloat16, sharp=True, seed=9)
    for c in comms:
        c.close()
    N = 32768
    rows = sample_rows(N, 40, seed=3, edges=[0, 1, 7, 8, 4095, 4096, N - 2, N - 1]).numpy()
    comms, _ = _check([(N, list(range(8)), "striped")], N, 32, 32, 128, torch.bfloat16, rows=rows)
    for c in comms:
        c.close()


def test_striped_store_layout_bit_exact():
    plan_list = [(512, [0, 1], "striped"), (512, [0, 1, 2, 3]), (1024, list(range(8)), "striped")]
    comms, (q, k, v) = _check(plan_list, 2048, 4, 2, 128, torch.bfloat16, seed=4)
    last_L, last_ranks = plan_list[-1][0], plan_list[-1][1]
    ext = plan_list + [(2 * len(last_ranks), last_ranks)]
    n, pos, _ = oracle.plan_stores(ext, len(plan_list))
    for i, inst in enumerate(last_ranks):
        st = comms[inst].kvstore()
        assert st.n == n[i]
        np.testing.assert_array_equal(st.pos[: st.n].cpu().numpy().astype(np.int64), pos[i])
        assert torch.equal(st.k[: st.n].cpu(), k[torch.as_tensor(pos[i])])
        assert torch.equal(st.v[: st.n].cpu(), v[torch.as_tensor(pos[i])])
    for c in comms:
        c.close()


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
@pytest.mark.parametrize("s,r,src,n,h", [(2, 0, 1, 64, 0), (4, 3, 1, 200, 77), (8, 2, 5, 130, 300), (8, 6, 6, 96, 0)])
def test_attention_fwd_strided_segments(dtype, s, r, src, n, h):
    """One ring step as a building block: q = stripe shard r, kv = h history rows + stripe shard
    src (positions j s + src), pos_stride = s — against oracle.attention on the positions."""
    D, Hq, Hkv = (128, 8, 2) if dtype == torch.bfloat16 else (64, 4, 4)
    C = 1000
    g = torch.Generator().manual_seed(s * 100 + r)
    q = torch.randn(n, Hq, D, generator=g).to(dtype)
    k = torch.randn(h + n, Hkv, D, generator=g).to(dtype)
    v = torch.randn(h + n, Hkv, D, generator=g).to(dtype)
    qpos = C + np.arange(n) * s + r
    kpos = np.concatenate([np.arange(h), C + np.arange(n) * s + src])  # history: positions < C
    m = n // 2
    seg = api.segments(n, m, C + r, C + r + m * s, h + n, h, m, C + src, C + src + m * s, pos_stride=s)
    out = torch.empty_like(q).cuda()
    lse = torch.empty(Hq, n, dtype=torch.float32, device="cuda")
    api.attention_fwd(q.cuda(), k.cuda(), v.cuda(), seg, out=out, lse=lse)
    torch.cuda.synchronize()
    o_ref, l_ref = oracle.attention(q.float().numpy(), qpos, k.float().numpy(), v.float().numpy(), kpos,
                                    1.0 / math.sqrt(D))
    ok = np.isfinite(l_ref)
    assert_out_close(out.float().cpu().numpy(), o_ref, dtype == torch.bfloat16)
    assert np.abs(lse.cpu().numpy()[ok] - l_ref[ok]).max() <= 1e-3
    assert np.all(np.isneginf(lse.cpu().numpy()[~ok]))


def test_striped_kv_transfer_bit_exact():
    Hkv, D, B, tp = 8, 128, 16, 8
    plan_list = [(512, [0, 1], "striped"), (512, [0, 1, 2, 3]), (1024, list(range(8)), "striped")]
    N = 2048
    _, k, v = qkv(N, 32, Hkv, D, torch.bfloat16, seed=5)
    plan = api.Plan(plan_list)
    n_logical = N // B
    nb = n_logical + 40
    bt = block_table(n_logical, nb, seed=7)
    kc = [torch.full((nb, B, Hkv // tp, D), 0x7FBF, dtype=torch.int16, device="cuda").view(torch.bfloat16)
          for _ in range(tp)]
    vc = [t.clone() for t in kc]
    dst = api.DecodeTarget(kc, vc, B, bt.cuda())
    comms = make_loopback_comms(plan, Hkv, D, torch.bfloat16)
    kd, vd = k.cuda(), v.cuda()
    for c, (L, ranks, *il) in enumerate(plan_list):
        C = plan.chunk_start(c)
        for r, inst in enumerate(ranks):
            ks = api.shard_gather(kd[C:C + L], len(ranks), r, plan.interleave[c])
            vs = api.shard_gather(vd[C:C + L], len(ranks), r, plan.interleave[c])
            api.kv_transfer_to_decode(ks, vs, api.SpGroup(comms[inst], plan, c), dst)
            assert api.kv_transfer_errors(comms[inst]) == 0
    torch.cuda.synchronize()
    ok = [np.full((nb, B, Hkv // tp, D), 0x7FBF, np.uint16) for _ in range(tp)]
    ov = [x.copy() for x in ok]
    oracle.paged_write(k.view(torch.int16).numpy().view(np.uint16), np.arange(N), tp, B, bt.numpy(), ok)
    oracle.paged_write(v.view(torch.int16).numpy().view(np.uint16), np.arange(N), tp, B, bt.numpy(), ov)
    for t in range(tp):
        assert np.array_equal(kc[t].cpu().view(torch.int16).numpy().view(np.uint16), ok[t])
        assert np.array_equal(vc[t].cpu().view(torch.int16).numpy().view(np.uint16), ov[t])
    for c in comms:
        c.close()
