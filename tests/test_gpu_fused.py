"""GPU parity of the fused ring (one launch walks every KV block of a rank's ring, O resident
in TMEM: cdsp_attention_fwd_blocks / the default bf16 path of cdsp_prefill_chunk) and of its
alternatives (multi-launch splits through the reserved accumulators, RING_STEPWISE, forced
arrival flags, the pre-staged control run) against the CPU oracle.

The reference is always the oracle's full causal attention over the unsharded prompt
(the ring covers every earlier key exactly once)."""
import math
import os

import numpy as np
import pytest
import torch

import oracle
from tolerances import assert_out_close
from cdsp_inputs import qkv, sample_rows
from paper_2511_06247_b200 import api
from paper_2511_06247_b200.driver import make_loopback_comms, run_plan_loopback

pytestmark = pytest.mark.gpu

TOL, LSE_TOL = 2e-2, 1e-3


def _ring_blocks(s, r, m, h, C, k_full, v_full):
    """The blocks ring rank r walks for a zigzag chunk of 2sm tokens at position C with h
    history rows per rank (history rows: positions < C, drawn from k_full[:C]): block k is src
    (r - k) mod s's store = its history part + its shard.  -> (ks, vs, segs)."""
    L = 2 * s * m
    ks, vs, segs = [], [], []
    for k in range(s):
        src = (r - k) % s
        hist = torch.arange(src * h, (src + 1) * h) if h else torch.zeros(0, dtype=torch.long)
        rows = torch.cat([hist, C + torch.arange(src * m, (src + 1) * m),
                          C + torch.arange((2 * s - 1 - src) * m, (2 * s - src) * m)])
        ks.append(k_full[rows].contiguous())
        vs.append(v_full[rows].contiguous())
        segs.append(api.segments(2 * m, m, C + r * m, C + (2 * s - 1 - r) * m, h + 2 * m, h, m,
                                 C + src * m, C + (2 * s - 1 - src) * m))
    qrows = torch.cat([C + torch.arange(r * m, (r + 1) * m), C + torch.arange((2 * s - 1 - r) * m, (2 * s - r) * m)])
    return ks, vs, segs, qrows


@pytest.mark.parametrize("s,m,h,Hq,Hkv,D", [
    (2, 128, 0, 4, 4, 128), (4, 96, 0, 4, 2, 128), (8, 64, 0, 2, 2, 128), (8, 160, 256, 4, 1, 128),
    (2, 300, 100, 2, 2, 64), (4, 128, 384, 8, 2, 64), (3, 70, 33, 2, 1, 128),
])
def test_blocks_one_launch_equals_full_causal(s, m, h, Hq, Hkv, D):
    """Every ring rank's s blocks in ONE launch = the rank's rows of full causal attention over
    history + chunk (history shards cover positions [0, C) exactly once)."""
    C = s * h
    N = C + 2 * s * m
    q, k, v = qkv(N, Hq, Hkv, D, torch.bfloat16, seed=s * 7 + m)
    o_ref, l_ref = oracle.causal_rows(q.float().numpy(), k.float().numpy(), v.float().numpy(), 1.0 / math.sqrt(D))
    for r in range(s):
        ks, vs, segs, qrows = _ring_blocks(s, r, m, h, C, k, v)
        qd = q[qrows].contiguous().cuda()
        out = torch.empty_like(qd)
        lse = torch.empty((Hq, 2 * m), dtype=torch.float32, device="cuda")
        api.attention_fwd_blocks(qd, [x.cuda() for x in ks], [x.cuda() for x in vs], segs, 0.0, api.ATTN_ONLY,
                                 out=out, lse=lse)
        torch.cuda.synchronize()
        err = np.abs(out.float().cpu().numpy() - o_ref[qrows.numpy()]).max()
        lerr = np.abs(lse.cpu().numpy() - l_ref[:, qrows.numpy()]).max()
        assert_out_close(out.float().cpu().numpy(), o_ref[qrows.numpy()], True, f"rank {r}")
        assert lerr <= LSE_TOL, (r, err, lerr)


@pytest.mark.parametrize("s,m,h,Hq,Hkv", [(8, 256, 0, 4, 4), (4, 384, 128, 4, 2), (2, 512, 0, 2, 1), (8, 512, 256, 8, 2)])
def test_blocks_split_units_with_scratch(s, m, h, Hq, Hkv):
    """ONLY mode with o_acc / lse_acc scratch: heavy (upper) units run as two sub-units merged
    in-kernel; every rank's rows still equal full causal attention (and the scratch-free launch)."""
    D = 128
    C = s * h
    N = C + 2 * s * m
    q, k, v = qkv(N, Hq, Hkv, D, torch.bfloat16, seed=s * 3 + m)
    o_ref, l_ref = oracle.causal_rows(q.float().numpy(), k.float().numpy(), v.float().numpy(), 1.0 / math.sqrt(D))
    for r in range(s):
        ks, vs, segs, qrows = _ring_blocks(s, r, m, h, C, k, v)
        qd = q[qrows].contiguous().cuda()
        ks, vs = [x.cuda() for x in ks], [x.cuda() for x in vs]
        acc = torch.full((2 * m, Hq, D), float("nan"), dtype=torch.float32, device="cuda")
        lacc = torch.full((Hq, 2 * m), float("nan"), dtype=torch.float32, device="cuda")
        out = torch.empty_like(qd)
        lse = torch.empty((Hq, 2 * m), dtype=torch.float32, device="cuda")
        for _ in range(3):  # repeated launches: the split counters are re-armed by each launch
            api.attention_fwd_blocks(qd, ks, vs, segs, 0.0, api.ATTN_ONLY, o_acc=acc, lse_acc=lacc, out=out, lse=lse)
        out2 = torch.empty_like(qd)
        api.attention_fwd_blocks(qd, ks, vs, segs, 0.0, api.ATTN_ONLY, out=out2)
        torch.cuda.synchronize()
        assert_out_close(out.float().cpu().numpy(), o_ref[qrows.numpy()], True, f"rank {r} split")
        assert np.abs(lse.cpu().numpy() - l_ref[:, qrows.numpy()]).max() <= LSE_TOL, r
        assert_out_close(out2.float().cpu().numpy(), o_ref[qrows.numpy()], True, f"rank {r} unsplit")


def test_blocks_first_last_chain_with_pdl():
    """The same union split into two launches (FIRST over blocks 0-1, LAST over 2-3, the LAST
    as a programmatic dependent) equals the one-launch result within tolerance."""
    s, m, h, Hq, Hkv, D = 4, 128, 128, 4, 2, 128
    C = s * h
    N = C + 2 * s * m
    q, k, v = qkv(N, Hq, Hkv, D, torch.bfloat16, seed=5)
    o_ref, l_ref = oracle.causal_rows(q.float().numpy(), k.float().numpy(), v.float().numpy(), 1.0 / math.sqrt(D))
    ks, vs, segs, qrows = _ring_blocks(s, 1, m, h, C, k, v)
    qd = q[qrows].contiguous().cuda()
    ks, vs = [x.cuda() for x in ks], [x.cuda() for x in vs]
    acc = torch.empty((2 * m, Hq, D), dtype=torch.float32, device="cuda")
    lacc = torch.empty((Hq, 2 * m), dtype=torch.float32, device="cuda")
    out = torch.empty_like(qd)
    lse = torch.empty_like(lacc)
    api.attention_fwd_blocks(qd, ks[:2], vs[:2], segs[:2], 0.0, api.ATTN_FIRST, o_acc=acc, lse_acc=lacc)
    api.attention_fwd_blocks(qd, ks[2:], vs[2:], segs[2:], 0.0, api.ATTN_LAST | api.ATTN_PDL, o_acc=acc, lse_acc=lacc,
                             out=out, lse=lse)
    torch.cuda.synchronize()
    assert_out_close(out.float().cpu().numpy(), o_ref[qrows.numpy()], True)
    assert np.abs(lse.cpu().numpy() - l_ref[:, qrows.numpy()]).max() <= LSE_TOL


def test_blocks_validation():
    q = torch.zeros(128, 2, 128, dtype=torch.bfloat16, device="cuda")
    kv = torch.zeros(128, 2, 128, dtype=torch.bfloat16, device="cuda")
    seg0 = api.causal_segments(128, 128)
    seg1 = api.causal_segments(128, 128, q_pos0=5)  # different query positions
    with pytest.raises(api.CdspError) as e:
        api.attention_fwd_blocks(q, [kv, kv], [kv, kv], [seg0, seg1], out=torch.empty_like(q))
    assert e.value.status == 2
    qf = q.float()
    with pytest.raises(api.CdspError) as e:  # fp32: one block per launch
        api.attention_fwd_blocks(qf, [kv.float()] * 2, [kv.float()] * 2, [seg0, seg0], out=torch.empty_like(qf))
    assert e.value.status == 8


def _loopback(plan_list, N, Hq, Hkv, D, dtype, options=0, reserve=True, rows=None, seed=0):
    q, k, v = qkv(N, Hq, Hkv, D, dtype, seed=seed)
    plan = api.Plan(plan_list)
    comms = make_loopback_comms(plan, Hkv, D, dtype, Hq=Hq if reserve else None)
    for c in comms:
        c.set_ring_options(options)
    out, lse = run_plan_loopback(q.cuda(), k.cuda(), v.cuda(), plan, comms=comms)
    torch.cuda.synchronize()
    o_ref, l_ref = oracle.causal_rows(q.float().numpy(), k.float().numpy(), v.float().numpy(), 1.0 / math.sqrt(D),
                                      rows=rows)
    o, l = out.float().cpu().numpy(), lse.cpu().numpy()
    if rows is not None:
        o, l = o[rows], l[:, rows]
    assert_out_close(o, o_ref, dtype == torch.bfloat16, str(plan_list))
    assert np.abs(l - l_ref).max() <= LSE_TOL, plan_list
    return comms, out, lse, (q, k, v), plan


RING_PLANS = [
    [(2048, [0, 1])],
    [(1024, [0, 1]), (1024, [0, 1, 2, 3]), (2048, list(range(8)))],
    [(512, [0]), (1536, [0, 1, 2, 3])],
]


@pytest.mark.parametrize("plan", RING_PLANS)
@pytest.mark.parametrize("options", [0, api.RING_STEPWISE, api.RING_GATE_FLAGS, api.RING_GATE_EVENTS])
def test_ring_modes_match_oracle(plan, options):
    N = sum(L for L, _ in plan)
    comms, *_ = _loopback(plan, N, 4, 2, 128, torch.bfloat16, options)
    for c in comms:
        c.check()  # no arrival-flag timeout
        c.close()


def test_ring_split_into_several_launches(monkeypatch):
    """A ring whose blocks exceed one launch's tile list runs as FIRST / MID / LAST launches
    merged in the reserved accumulators (budget shrunk to 6 tiles by the test knob)."""
    monkeypatch.setenv("CDSP_MAX_TILES", "6")
    comms, *_ = _loopback([(1024, [0, 1]), (2048, list(range(8)))], 3072, 4, 2, 128, torch.bfloat16)
    for c in comms:
        c.close()


def test_ring_grouped_by_l2_budget(monkeypatch):
    """With accumulators reserved, the ring's blocks are grouped into launches whose per-KV-head
    K / V fits the L2 budget (forced to 1 MB here: one launch per block, merged in fp32)."""
    monkeypatch.setenv("CDSP_RING_L2_MB", "1")
    import subprocess, sys  # the budget is read once per process: run the check in a fresh one
    code = ("import sys; sys.path.insert(0, 'tests'); import test_gpu_fused as t; "
            "t._loopback([(2048, [0, 1]), (6144, list(range(8)))], 8192, 4, 2, 128, t.torch.bfloat16)")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, "-c", code], cwd=root, capture_output=True, text=True, timeout=600,
                         env=dict(os.environ, CDSP_RING_L2_MB="1"))
    assert out.returncode == 0, out.stderr[-3000:]


def test_multi_launch_ring_needs_reserved_accumulators():
    plan = api.Plan([(512, [0, 1])])
    comms = make_loopback_comms(plan, 2, 64, torch.float32)  # no Hq: nothing reserved
    q, k, v = (t.cuda() for t in qkv(512, 2, 2, 64, torch.float32))
    with pytest.raises(api.CdspError) as e:
        run_plan_loopback(q, k, v, plan, comms=comms)
    assert e.value.status == 5
    for c in comms:
        c.close()


def test_control_run_reuses_prestaged_blocks():
    """RING_CONTROL: no pulls — a second call with the same inputs over the blocks the first
    call pulled reproduces the first call's output (up to the order in which split sub-units
    merge, which is decided at run time: same tolerance as against the oracle)."""
    plan_list = [(4096, list(range(4)))]
    comms, out1, lse1, (q, k, v), plan = _loopback(plan_list, 4096, 4, 4, 128, torch.bfloat16, 0)
    for c in comms:
        c.set_ring_options(api.RING_CONTROL)
    out2, lse2 = run_plan_loopback(q.cuda(), k.cuda(), v.cuda(), plan, comms=comms)
    torch.cuda.synchronize()
    o_ref, l_ref = oracle.causal_rows(q.float().numpy(), k.float().numpy(), v.float().numpy(), 1.0 / math.sqrt(128))
    assert_out_close(out2.float().cpu().numpy(), o_ref, True, "control run")
    assert np.abs(lse2.cpu().numpy() - l_ref).max() <= LSE_TOL
    assert (out1.float() - out2.float()).abs().max().item() <= 2 ** -6  # one bf16 ulp at |o| < 2
    for c in comms:
        c.close()


def test_m2_shape_sp8_fused_and_flags_sampled():
    """configs[1] (32K MHA 32/32, d=128, one chunk at SP=8): fused ring, default and forced
    arrival flags, on sampled rows (shard edges included)."""
    N = 32768
    rows = sample_rows(N, 32, seed=9, edges=[0, 2047, 2048, 4095, 4096, 30719, 30720, N - 1]).numpy()
    for opt in (0, api.RING_GATE_FLAGS):
        comms, *_ = _loopback([(N, list(range(8)))], N, 32, 32, 128, torch.bfloat16, opt, rows=rows)
        for c in comms:
            c.check()
            c.close()


_PACING_CODE = """
import sys, math, json
sys.path.insert(0, 'tests')
import numpy as np, torch, oracle
from tolerances import assert_out_close
from cdsp_inputs import qkv, sample_rows
from paper_2511_06247_b200 import api
from paper_2511_06247_b200.driver import make_loopback_comms, run_plan_loopback
N, Hq, Hkv, D = 40960, 32, 8, 128
plan = api.Plan([(N, list(range(8)))])
q, k, v = qkv(N, Hq, Hkv, D, torch.bfloat16, seed=5)
comms = make_loopback_comms(plan, Hkv, D, torch.bfloat16, Hq=Hq)
for c in comms:
    c.set_ring_options(api.RING_GATE_FLAGS)
    c.profile(True)
out, lse = run_plan_loopback(q.cuda(), k.cuda(), v.cuda(), plan, comms=comms)
torch.cuda.synchronize()
n = max(c.profile_read()[1] for c in comms)
rows = sample_rows(N, 24, seed=1, edges=[0, N - 1]).numpy()
o_ref, l_ref = oracle.causal_rows(q.float().numpy(), k.float().numpy(), v.float().numpy(), 1.0 / math.sqrt(D), rows=rows)
assert_out_close(out.float().cpu().numpy()[rows], o_ref, True, 'paced ring')
assert np.abs(lse.cpu().numpy()[:, rows] - l_ref).max() <= 1e-3
print(json.dumps({'launches_per_rank': n}))
"""


@pytest.mark.parametrize("link_gbs,grouped", [(None, False), ("150", True)])
def test_ring_pull_pacing(link_gbs, grouped):
    """Flag-gated SP = 8 ring of a 40K-token chunk (8.6 waves of units per rank): at the default
    link rate the pulls are short against the compute and the ring stays ONE fused launch; at
    150 GB/s (CDSP_RING_LINK_GBS) the first wave of a fused launch would wait out most of the
    pulls, so the blocks are grouped into several launches merged in fp32 — either way the
    result matches the oracle."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ)
    env.pop("CDSP_RING_LINK_GBS", None)
    if link_gbs:
        env["CDSP_RING_LINK_GBS"] = link_gbs
    out = subprocess.run([sys.executable, "-c", _PACING_CODE], cwd=root, capture_output=True, text=True, timeout=900,
                         env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    n = json.loads([l for l in out.stdout.splitlines() if l.startswith("{")][-1])["launches_per_rank"]
    assert (n > 1) == grouped, n
