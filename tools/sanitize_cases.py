"""Tiny invocations of every kernel of the library, for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck): tcgen05 attention (2-SM PAIR at D=128, 1-SM at D=64) in every mode incl.
a FIRST / MID / LAST chain with programmatic dependent launch, the fused multi-block launch with
split units, the fp32 FFMA kernel, the LSE merge, zigzag / striped copies, store append, paged
scatter, decode, and a loopback SP=2 ring through cdsp_prefill_chunk (events and arrival flags).
usage: compute-sanitizer --tool <t> python tools/sanitize_cases.py"""
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from cdsp_inputs import block_table, qkv  # noqa: E402
from paper_2511_06247_b200 import api  # noqa: E402
from paper_2511_06247_b200.driver import make_loopback_comms, run_plan_loopback  # noqa: E402

dev = "cuda"
for D, N, Hq, Hkv in ((128, 300, 2, 1), (64, 200, 2, 2)):
    q, k, v = (t.to(dev) for t in qkv(N, Hq, Hkv, D, torch.bfloat16, seed=1))
    out = torch.empty_like(q)
    lse = torch.empty(Hq, N, device=dev)
    api.attention_fwd(q, k, v, api.causal_segments(N, N), 0.0, api.ATTN_ONLY, out=out, lse=lse)
    acc = torch.empty(N, Hq, D, device=dev)
    lacc = torch.empty(Hq, N, device=dev)
    half = N // 2
    seg_a = api.segments(N, N, 0, 0, half, 0, half, 0, 0)            # keys [0, half)
    seg_b = api.segments(N, N, 0, 0, N - half, 0, N - half, half, 0)  # keys [half, N)
    kb, vb = k[half:].contiguous(), v[half:].contiguous()
    api.attention_fwd(q, k, v, seg_a, 0.0, api.ATTN_FIRST, o_acc=acc, lse_acc=lacc)
    api.attention_fwd(q, kb, vb, seg_b, 0.0, api.ATTN_MID | api.ATTN_PDL, o_acc=acc, lse_acc=lacc)
    api.attention_fwd(q, k, v, api.segments(N, N, 0, 0, 0, 0, 0, 0, 0), 0.0, api.ATTN_LAST | api.ATTN_PDL,
                      o_acc=acc, lse_acc=lacc, out=out, lse=lse)
    # fused blocks (+ split units through the scratch)
    api.attention_fwd_blocks(q, [k, kb], [v, vb], [seg_a, seg_b], 0.0, api.ATTN_ONLY, out=out, lse=lse,
                             o_acc=acc, lse_acc=lacc)
    torch.cuda.synchronize()
# fp32 FFMA kernel
q, k, v = (t.to(dev) for t in qkv(130, 2, 1, 64, torch.float32, seed=2))
api.attention_fwd(q, k, v, api.causal_segments(130, 130), 0.0, api.ATTN_ONLY, out=torch.empty_like(q))
# merge
parts = [torch.randn(70, 3, 64, device=dev) for _ in range(3)]
lses = [torch.randn(3, 70, device=dev) for _ in range(3)]
lses[1][0, :5] = -math.inf
api.lse_merge(parts, lses, torch.empty(70, 3, 64, dtype=torch.bfloat16, device=dev), torch.empty(3, 70, device=dev))
# copies
full = torch.randn(256, 2, 64, device=dev).to(torch.bfloat16)
sh = api.zigzag_gather(full, 4, 1)
api.zigzag_scatter(sh, 4, 1, torch.empty_like(full))
st = api.striped_gather(full, 4, 2)
api.striped_scatter(st, 4, 2, torch.empty_like(full))
api.zigzag_map_device(256, 4)
# ring + store append + paged scatter + decode
for opts in (0, api.RING_GATE_FLAGS):
    plan = api.Plan([(256, [0]), (512, [0, 1])])
    q, k, v = (t.to(dev) for t in qkv(768, 4, 2, 128, torch.bfloat16, seed=3))
    comms = make_loopback_comms(plan, 2, 128, torch.bfloat16, Hq=4)
    for c in comms:
        c.set_ring_options(opts)
    run_plan_loopback(q, k, v, plan, comms=comms)
    torch.cuda.synchronize()
    for c in comms:
        c.close()
plan = api.Plan([(256, [0])])
comm = api.Comm(0, 1, 0, 256, 2, 128, torch.bfloat16)
k = torch.randn(256, 2, 128, device=dev).to(torch.bfloat16)
B = 16
bt = block_table(16, 24, seed=7).to(dev)
kc = [torch.zeros(24, B, 1, 128, dtype=torch.bfloat16, device=dev) for _ in range(2)]
vc = [torch.zeros_like(x) for x in kc]
tgt = api.DecodeTarget(kc, vc, B, bt)
api.kv_transfer_to_decode(k, k, api.SpGroup(comm, plan, 0), tgt)
qd = torch.randn(1, 2, 128, device=dev).to(torch.bfloat16)
api.decode_attention(qd, tgt, 0, 1, 256)   # TMA-fed kernel (B >= 16), slice merge over its splits
api.decode_attention(qd, tgt, 0, 1, 250)   # ragged last page (V rows past the range zeroed)
torch.cuda.synchronize()
comm.close()
# decode with 8-token pages (cp.async kernel) and in fp32 (FFMA kernel)
for dt, B8 in ((torch.bfloat16, 8), (torch.float32, 16)):
    plan = api.Plan([(512, [0])])
    comm = api.Comm(0, 1, 0, 512, 1, 128, dt)
    k = torch.randn(512, 1, 128, device=dev).to(dt)
    bt = block_table(512 // B8, 512 // B8 + 4, seed=5).to(dev)
    kc = [torch.zeros(512 // B8 + 4, B8, 1, 128, dtype=dt, device=dev)]
    vc = [torch.zeros_like(kc[0])]
    tgt = api.DecodeTarget(kc, vc, B8, bt)
    api.kv_transfer_to_decode(k, k, api.SpGroup(comm, plan, 0), tgt)
    api.decode_attention(torch.randn(1, 4, 128, device=dev).to(dt), tgt, 0, 1, 509)
    torch.cuda.synchronize()
    comm.close()
# prefill + transfer in one call (scatter on the communicator's transfer stream)
plan = api.Plan([(256, [0])])
comm = api.Comm(0, 1, 0, 256, 2, 128, torch.bfloat16)
q, k, v = (t.to(dev) for t in qkv(256, 4, 2, 128, torch.bfloat16, seed=4))
bt = block_table(16, 20, seed=2).to(dev)
kc = [torch.zeros(20, 16, 1, 128, dtype=torch.bfloat16, device=dev) for _ in range(2)]
vc = [torch.zeros_like(x) for x in kc]
api.prefill_chunk_transfer(q, k, v, comm.kvstore(), api.SpGroup(comm, plan, 0), api.DecodeTarget(kc, vc, 16, bt))
torch.cuda.synchronize()
comm.close()
print("sanitize cases done")
