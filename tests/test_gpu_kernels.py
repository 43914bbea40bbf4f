"""GPU parity of the individual kernels (through the C ABI) against the CPU oracle.

Tolerances (north_star): attention out max-abs 2e-2 (bf16 path) / 1e-4 (fp32 path), LSE
1e-3; partition maps and KV layout bit-exact."""
import math

import numpy as np
import pytest
import torch

import oracle
from tolerances import assert_out_close
from cdsp_inputs import qkv, sample_rows
from paper_2511_06247_b200 import api

pytestmark = pytest.mark.gpu

TOL = {torch.bfloat16: 2e-2, torch.float32: 1e-4}
LSE_TOL = 1e-3


def _np(x):
    return x.detach().float().cpu().numpy()


def _check(out, lse, o_ref, l_ref, dtype, what=""):
    err = np.abs(_np(out).astype(np.float64) - o_ref).max() if o_ref.size else 0.0
    fin = np.isfinite(l_ref)
    lerr = np.abs(_np(lse).astype(np.float64)[fin] - l_ref[fin])
    lerr = lerr.max() if fin.any() else 0.0
    assert np.array_equal(np.isfinite(_np(lse)), np.isfinite(l_ref)), f"{what}: -inf pattern differs"
    assert_out_close(_np(out), o_ref, dtype == torch.bfloat16, what)
    assert lerr <= LSE_TOL, f"{what}: lse max-abs {lerr:.3e}"
    return err, lerr


CASES = [
    (1, 2, 2, 64, torch.bfloat16), (77, 2, 2, 128, torch.bfloat16), (128, 4, 4, 128, torch.bfloat16),
    (300, 4, 1, 128, torch.bfloat16), (513, 8, 2, 64, torch.bfloat16), (1000, 2, 2, 128, torch.bfloat16),
    (1, 2, 1, 64, torch.float32), (100, 4, 4, 64, torch.float32), (257, 2, 1, 128, torch.float32),
    (700, 3, 3, 64, torch.bfloat16),
]


@pytest.mark.parametrize("N,Hq,Hkv,D,dtype", CASES)
@pytest.mark.parametrize("sharp", [False, True])
def test_causal_attention_all_rows(N, Hq, Hkv, D, dtype, sharp):
    q, k, v = qkv(N, Hq, Hkv, D, dtype, seed=N + D, sharp=sharp)
    scale = 1.0 / math.sqrt(D)
    qd, kd, vd = q.cuda(), k.cuda(), v.cuda()
    out = torch.empty_like(qd)
    lse = torch.empty((Hq, N), dtype=torch.float32, device="cuda")
    api.attention_fwd(qd, kd, vd, api.causal_segments(N, N), scale, api.ATTN_ONLY, out=out, lse=lse)
    torch.cuda.synchronize()
    o_ref, l_ref = oracle.causal_rows(q.float().numpy(), k.float().numpy(), v.float().numpy(), scale)
    _check(out, lse, o_ref, l_ref, dtype, f"N={N} Hq={Hq} Hkv={Hkv} D={D} {dtype}")


def _zigzag_block_case(s, r, src, m, h, Hq, Hkv, D, dtype, C=1000, seed=0):
    """Q = rank r's shard of a chunk at C; KV = src's history (h rows) + src's shard."""
    L = 2 * s * m
    q, k, v = qkv(L, Hq, Hkv, D, dtype, seed=seed)
    hk, hv = qkv(max(h, 1), Hkv, Hkv, D, dtype, seed=seed + 50)[1:]
    hk, hv = hk[:h], hv[:h]
    pos = oracle.rank_positions(L, s, C)
    qs, ks, vs = q[pos[r] - C], k[pos[src] - C], v[pos[src] - C]
    kk = torch.cat([hk, ks]).contiguous()
    vv = torch.cat([hv, vs]).contiguous()
    kpos = np.concatenate([np.arange(h) + C - h - 7, pos[src]])
    seg = api.segments(2 * m, m, C + r * m, C + (2 * s - 1 - r) * m, h + 2 * m, h, m, C + src * m,
                       C + (2 * s - 1 - src) * m)
    return qs.contiguous(), kk, vv, pos[r], kpos, seg


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
@pytest.mark.parametrize("s,r,src,m,h", [(2, 0, 0, 64, 0), (2, 1, 0, 96, 50), (4, 1, 3, 130, 257),
                                         (8, 5, 2, 128, 384), (8, 2, 6, 40, 1), (4, 3, 3, 200, 130)])
def test_block_with_history_and_zigzag_segments(dtype, s, r, src, m, h):
    Hq, Hkv, D = (4, 2, 128) if dtype == torch.bfloat16 else (2, 2, 64)
    qs, kk, vv, qpos, kpos, seg = _zigzag_block_case(s, r, src, m, h, Hq, Hkv, D, dtype, seed=s * 10 + r)
    scale = 1.0 / math.sqrt(D)
    out = torch.empty_like(qs).cuda()
    lse = torch.empty((Hq, 2 * m), dtype=torch.float32, device="cuda")
    api.attention_fwd(qs.cuda(), kk.cuda(), vv.cuda(), seg, scale, api.ATTN_ONLY, out=out, lse=lse)
    torch.cuda.synchronize()
    o_ref, l_ref = oracle.attention(qs.float().numpy(), qpos, kk.float().numpy(), vv.float().numpy(), kpos, scale)
    _check(out, lse, o_ref, l_ref, dtype, f"s={s} r={r} src={src} m={m} h={h}")


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
def test_merge_modes_chain_equals_single_block(dtype):
    """FIRST / MID / LAST over three KV blocks == ONLY over their union (R3 in the epilogue)."""
    N, Hq, Hkv, D = 640, 4, 4, 128 if dtype == torch.bfloat16 else 64
    q, k, v = (t.cuda() for t in qkv(N, Hq, Hkv, D, dtype, seed=3))
    scale = 1.0 / math.sqrt(D)
    cuts = [0, 200, 300, N]
    o_acc = torch.empty((N, Hq, D), dtype=torch.float32, device="cuda")
    l_acc = torch.empty((Hq, N), dtype=torch.float32, device="cuda")
    out = torch.empty_like(q)
    lse = torch.empty((Hq, N), dtype=torch.float32, device="cuda")
    modes = [api.ATTN_FIRST, api.ATTN_MID, api.ATTN_LAST]
    for (a, b), mode in zip(zip(cuts[:-1], cuts[1:]), modes):
        seg = api.segments(N, N, 0, 0, b - a, 0, b - a, a, 0)
        api.attention_fwd(q, k[a:b].contiguous(), v[a:b].contiguous(), seg, scale, mode, o_acc, l_acc, out, lse)
    torch.cuda.synchronize()
    o_ref, l_ref = oracle.causal_rows(_np(q), _np(k), _np(v), scale)
    _check(out, lse, o_ref, l_ref, dtype, "merge chain")


def test_fully_masked_block_is_identity():
    """A block invisible to every query (src > r, first half) leaves the accumulator exact."""
    m, Hq, D = 128, 2, 128
    q = torch.randn(2 * m, Hq, D, device="cuda").to(torch.bfloat16)
    k = torch.randn(2 * m, Hq, D, device="cuda").to(torch.bfloat16)
    o_acc = torch.randn(2 * m, Hq, D, device="cuda")
    l_acc = torch.randn(Hq, 2 * m, device="cuda")
    o0, l0 = o_acc.clone(), l_acc.clone()
    seg = api.segments(2 * m, 2 * m, 0, 0, 2 * m, 0, 2 * m, 10000, 10000)  # keys all in the future
    api.attention_fwd(q, k, k, seg, 0.1, api.ATTN_MID, o_acc, l_acc)
    torch.cuda.synchronize()
    assert torch.equal(l_acc, l0)
    assert (o_acc - o0).abs().max().item() <= 1e-6


@pytest.mark.parametrize("n", [1, 2, 3, 8])
@pytest.mark.parametrize("D", [64, 128])
def test_lse_merge_kernel(n, D):
    T, H = 333, 3
    g = torch.Generator().manual_seed(n * D)
    parts = [torch.randn(T, H, D, generator=g) for _ in range(n)]
    lses = [torch.randn(H, T, generator=g) * 4 for _ in range(n)]
    lses[0][0, :10] = float("-inf")
    if n > 1:
        for l in lses:
            l[1, 5] = float("-inf")  # a row with every part empty
    out = torch.empty(T, H, D, device="cuda")
    lse = torch.empty(H, T, device="cuda")
    api.lse_merge([p.cuda() for p in parts], [l.cuda() for l in lses], out, lse)
    outb = torch.empty(T, H, D, device="cuda", dtype=torch.bfloat16)
    api.lse_merge([p.cuda() for p in parts], [l.cuda() for l in lses], outb)
    torch.cuda.synchronize()
    o_ref, l_ref = oracle.lse_merge([p.double().numpy() for p in parts], [l.double().numpy() for l in lses])
    assert np.abs(_np(out) - o_ref).max() <= 1e-5
    fin = np.isfinite(l_ref)
    assert np.array_equal(np.isfinite(_np(lse)), fin)
    assert np.abs(_np(lse)[fin] - l_ref[fin]).max() <= 1e-5
    assert not np.isnan(_np(out)).any()
    assert_out_close(_np(outb), o_ref, True)


@pytest.mark.parametrize("s", [1, 2, 4, 8])
@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
def test_zigzag_gather_scatter_bit_exact(s, dtype):
    L, H, D = 2 * s * 37, 3, 64
    full = torch.randn(L, H, D, device="cuda").to(dtype)
    tr, ts = oracle.zigzag_map(L, s)
    back = torch.zeros_like(full)
    for r in range(s):
        sh = api.zigzag_gather(full, s, r)
        idx = np.nonzero(tr == r)[0]
        expect = torch.empty_like(sh)
        expect[torch.as_tensor(ts[idx], device="cuda").long()] = full[torch.as_tensor(idx, device="cuda")]
        assert torch.equal(sh, expect)
        api.zigzag_scatter(sh, s, r, back)
    torch.cuda.synchronize()
    assert torch.equal(back, full)


@pytest.mark.parametrize("s", [1, 2, 4, 8])
def test_device_zigzag_map_bit_exact(s):
    L = 2 * s * 1000
    tr, ts = api.zigzag_map_device(L, s)
    otr, ots = oracle.zigzag_map(L, s)
    assert np.array_equal(tr.cpu().numpy(), otr) and np.array_equal(ts.cpu().numpy(), ots)


def test_bench_config_sampled_rows():
    """BASELINE configs[1] shape (7B MHA, 32 heads, d=128, 32K) at SP=1 through
    cdsp_prefill_chunk, the launch the bench times; sampled rows incl. tile edges."""
    N, Hq, Hkv, D = 32768, 32, 32, 128
    q, k, v = qkv(N, Hq, Hkv, D, torch.bfloat16, seed=0)
    plan = api.Plan([(N, [0])])
    comm = api.Comm(0, 1, 0, N, Hkv, D, torch.bfloat16)
    out = torch.empty(N, Hq, D, dtype=torch.bfloat16, device="cuda")
    lse = torch.empty(Hq, N, dtype=torch.float32, device="cuda")
    api.prefill_chunk(q.cuda(), k.cuda(), v.cuda(), comm.kvstore(), api.SpGroup(comm, plan, 0), 0.0, out, lse)
    torch.cuda.synchronize()
    rows = sample_rows(N, 48, seed=1, edges=[0, 1, 127, 128, 255, 256, 16383, 16384, N - 129, N - 1]).numpy()
    o_ref, l_ref = oracle.causal_rows(q.float().numpy(), k.float().numpy(), v.float().numpy(),
                                      1.0 / math.sqrt(D), rows=rows)
    _check(out[torch.as_tensor(rows, device="cuda")], lse[:, torch.as_tensor(rows, device="cuda")], o_ref, l_ref,
           torch.bfloat16, "32K sampled")
    comm.close()


# ---- persistent 2-SM kernel edge cases: units with no visible key, the unit counter ring, capacity
def _empty_half_case(mode, dtype, m=200, Hq=4, Hkv=2, D=128, seed=11):
    """Query rows of segment 0 (positions 0..m-1) see no key (keys at 5000..), segment 1 rows
    (positions 20000..) see all: whole 128-row units have no visible tile."""
    q, k, v = (t.cuda() for t in qkv(2 * m, Hq, Hkv, D, dtype, seed=seed))
    seg = api.segments(2 * m, m, 0, 20000, 2 * m, 0, 2 * m, 5000, 0)
    qpos = np.concatenate([np.arange(m), 20000 + np.arange(m)])
    kpos = 5000 + np.arange(2 * m)
    return q, k, v, seg, qpos, kpos


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
def test_rows_without_keys_only_mode(dtype):
    D = 128 if dtype == torch.bfloat16 else 64
    q, k, v, seg, qpos, kpos = _empty_half_case(api.ATTN_ONLY, dtype, D=D)
    scale = 1.0 / math.sqrt(D)
    out = torch.full_like(q, 7.0)
    lse = torch.full((q.shape[1], q.shape[0]), 7.0, dtype=torch.float32, device="cuda")
    api.attention_fwd(q, k, v, seg, scale, api.ATTN_ONLY, out=out, lse=lse)
    torch.cuda.synchronize()
    o_ref, l_ref = oracle.attention(_np(q), qpos, _np(k), _np(v), kpos, scale)
    o_ref = np.where(np.isfinite(l_ref).T[:, :, None], o_ref, 0.0)  # no key: out 0, lse -inf (R3, R16)
    _check(out, lse, o_ref, l_ref, dtype, "ONLY, rows without keys")


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
def test_rows_without_keys_first_and_last_modes(dtype):
    """FIRST writes (0, -inf) for rows without keys; LAST merges (R3): such rows get the
    accumulator unchanged (rounded to the output dtype), the others merge with the block."""
    D = 128 if dtype == torch.bfloat16 else 64
    q, k, v, seg, qpos, kpos = _empty_half_case(api.ATTN_LAST, dtype, D=D, seed=12)
    n, Hq = q.shape[0], q.shape[1]
    scale = 1.0 / math.sqrt(D)
    o_ref, l_ref = oracle.attention(_np(q), qpos, _np(k), _np(v), kpos, scale)
    o_blk = np.where(np.isfinite(l_ref).T[:, :, None], o_ref, 0.0)
    # FIRST
    o_acc = torch.full((n, Hq, D), 3.0, dtype=torch.float32, device="cuda")
    l_acc = torch.full((Hq, n), 3.0, dtype=torch.float32, device="cuda")
    api.attention_fwd(q, k, v, seg, scale, api.ATTN_FIRST, o_acc, l_acc)
    torch.cuda.synchronize()
    assert np.abs(_np(o_acc) - o_blk).max() <= 1e-2
    assert np.array_equal(np.isfinite(_np(l_acc)), np.isfinite(l_ref))
    fin = np.isfinite(l_ref)
    assert np.abs(_np(l_acc)[fin] - l_ref[fin]).max() <= LSE_TOL
    # LAST over a random accumulator
    g = torch.Generator().manual_seed(5)
    acc = torch.randn((n, Hq, D), generator=g).cuda()
    lacc = torch.randn((Hq, n), generator=g).cuda()
    out = torch.empty_like(q)
    lse = torch.empty((Hq, n), dtype=torch.float32, device="cuda")
    api.attention_fwd(q, k, v, seg, scale, api.ATTN_LAST, acc.clone(), lacc.clone(), out, lse)
    torch.cuda.synchronize()
    m_ref, ml_ref = oracle.lse_merge([_np(acc).astype(np.float64), o_blk], [_np(lacc).astype(np.float64), l_ref])
    _check(out, lse, m_ref, ml_ref, dtype, "LAST, rows without keys")
    rows0 = slice(0, n // 2)  # segment 0: no key -> exactly the accumulator, rounded once
    assert torch.equal(out[rows0], acc[rows0].to(dtype))
    assert torch.equal(lse[:, rows0], lacc[:, rows0])


def test_unit_counter_ring_many_launches():
    """> 4096 back-to-back launches cycle every slot of the persistent kernel's unit-counter
    ring (each launch's last CTA re-arms its slot); results stay identical."""
    N, Hq, D = 384, 2, 128
    q, k, v = (t.cuda() for t in qkv(N, Hq, Hq, D, torch.bfloat16, seed=21))
    ref = torch.empty_like(q)
    api.attention_fwd(q, k, v, api.causal_segments(N, N), 0.0, api.ATTN_ONLY, out=ref)
    out = torch.empty_like(q)
    for _ in range(4200):
        api.attention_fwd(q, k, v, api.causal_segments(N, N), 0.0, api.ATTN_ONLY, out=out)
    torch.cuda.synchronize()
    assert torch.equal(out, ref)


def test_kv_block_capacity_error():
    """One block-attention launch takes at most 4096 KV tiles (512K keys): more is
    CDSP_ERR_CAPACITY before anything is launched."""
    nkv = 4096 * 128 + 1
    q = torch.zeros((128, 1, 128), dtype=torch.bfloat16, device="cuda")
    k = torch.zeros((nkv, 1, 128), dtype=torch.bfloat16, device="cuda")
    with pytest.raises(api.CdspError) as ei:
        api.attention_fwd(q, k, k, api.causal_segments(128, nkv, q_pos0=nkv - 128), 0.0, api.ATTN_ONLY,
                          out=torch.empty_like(q))
    assert ei.value.status == 5


def test_back_to_back_merge_chain_programmatic_launch():
    """FIRST, 6 x MID, LAST over 8 KV blocks of one 16K causal prompt, launched back to back on
    one stream: each MID / LAST grid is a programmatic dependent of the previous one (it starts
    its main loop under the predecessor's tail and touches the accumulator after
    griddepcontrol.wait).  Sampled rows vs the oracle; GQA 32/8 so units are many and long."""
    N, Hq, Hkv, D = 16384, 16, 4, 128
    q, k, v = (t.cuda() for t in qkv(N, Hq, Hkv, D, torch.bfloat16, seed=31))
    scale = 1.0 / math.sqrt(D)
    o_acc = torch.empty((N, Hq, D), dtype=torch.float32, device="cuda")
    l_acc = torch.empty((Hq, N), dtype=torch.float32, device="cuda")
    out = torch.empty_like(q)
    lse = torch.empty((Hq, N), dtype=torch.float32, device="cuda")
    cuts = [i * N // 8 for i in range(9)]
    blocks = [(k[a:b].contiguous(), v[a:b].contiguous()) for a, b in zip(cuts[:-1], cuts[1:])]
    torch.cuda.synchronize()
    for i, ((a, b), (kb, vb)) in enumerate(zip(zip(cuts[:-1], cuts[1:]), blocks)):
        mode = api.ATTN_FIRST if i == 0 else api.ATTN_LAST if i == 7 else api.ATTN_MID
        seg = api.segments(N, N, 0, 0, b - a, 0, b - a, a, 0)
        api.attention_fwd(q, kb, vb, seg, scale, mode, o_acc, l_acc, out, lse)
    torch.cuda.synchronize()
    rows = sample_rows(N, 256, seed=5, edges=[0, 127, 128, 2047, 2048, N - 1])
    o_ref, l_ref = oracle.causal_rows(_np(q), _np(k), _np(v), scale, rows=rows.numpy())
    _check(out[rows], lse[:, rows], o_ref, l_ref, torch.bfloat16, "back-to-back chain")


def test_kv_block_at_capacity_512k_keys():
    """One launch over exactly 4096 KV tiles (512K keys, the per-unit tile list at full length):
    the last 200 query rows of a 512K causal prompt, sampled vs the oracle."""
    nkv, nq, Hq, Hkv, D = 4096 * 128, 200, 2, 1, 128
    q, k, v = (t.cuda() for t in qkv(nkv, Hq, Hkv, D, torch.bfloat16, seed=41))
    qs = q[nkv - nq:].contiguous()
    out = torch.empty_like(qs)
    lse = torch.empty((Hq, nq), dtype=torch.float32, device="cuda")
    scale = 1.0 / math.sqrt(D)
    api.attention_fwd(qs, k, v, api.causal_segments(nq, nkv, q_pos0=nkv - nq), scale, api.ATTN_ONLY,
                      out=out, lse=lse)
    torch.cuda.synchronize()
    rows = sample_rows(nq, 24, seed=3, edges=[0, 127, 128, nq - 1])
    o_ref, l_ref = oracle.causal_rows(_np(q), _np(k), _np(v), scale, rows=(rows + nkv - nq).numpy())
    _check(out[rows], lse[:, rows], o_ref, l_ref, torch.bfloat16, "512K keys")


def test_one_sm_kernel_d128_subprocess():
    """CDSP_ATTN_1SM=1 (read once per process) runs D = 128 on the 1-SM kernel instead of CTA
    pairs (the measurement control of DESIGN 6.1): a ragged causal launch, every row vs the
    oracle, in a fresh process."""
    import os
    import subprocess
    import sys
    code = r'''
import math, numpy as np, torch, oracle
from cdsp_inputs import qkv
from paper_2511_06247_b200 import api
N, Hq, Hkv, D = 1500, 4, 2, 128
q, k, v = qkv(N, Hq, Hkv, D, torch.bfloat16, seed=77)
s = 1.0 / math.sqrt(D)
out = torch.empty_like(q.cuda()); lse = torch.empty((Hq, N), dtype=torch.float32, device="cuda")
api.attention_fwd(q.cuda(), k.cuda(), v.cuda(), api.causal_segments(N, N), s, api.ATTN_ONLY, out=out, lse=lse)
torch.cuda.synchronize()
o_ref, l_ref = oracle.causal_rows(q.float().numpy(), k.float().numpy(), v.float().numpy(), s)
print("ERR", float(np.abs(out.float().cpu().numpy() - o_ref).max()), float(np.abs(lse.cpu().numpy() - l_ref).max()))
'''
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, CDSP_ATTN_1SM="1", PYTHONPATH=root)
    r = subprocess.run([sys.executable, "-c", code], env=env, cwd=root, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    err, lerr = [float(x) for x in [l for l in r.stdout.splitlines() if l.startswith("ERR")][0].split()[1:]]
    assert err <= 2e-2 and lerr <= 1e-3, (err, lerr)
