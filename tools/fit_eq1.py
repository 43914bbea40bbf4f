"""Eq. (1) of the paper (§5.1) fitted on B200: T_s(C, L) = a + b L + c C L + d L^2 for
ONE attention layer of the LLaMA3-8B shape (GQA 32/8, d=128, bf16) through this library.

  s = 1: measured through cdsp_prefill_chunk itself (a plan [(C, [0]), (L, [0])]: the timed call
         is chunk 1 — store append + attention over C history rows + the L-token chunk);
  s > 1: PROXY on one GPU — every ring rank's fused launch (cdsp_attention_fwd_blocks over its s
         blocks: C/s history rows + the 2m-row shard of each source, peer blocks resident) is
         timed on its own, and the chunk's latency is the slowest rank's (ranks run in parallel
         on s GPUs; the ring pulls, hidden under compute on NVLink, are not in the number).

Each (s, C, L) point: median of --iters timed calls after warm-up (CUDA events).  The fit is
cdsp_fit_latency_model (scaled Householder least squares); coefficients, samples and the relative
residuals go to one JSON document (profiles/r02_eq1_fit.json).
usage: python tools/fit_eq1.py [--iters 5] [--out profiles/r02_eq1_fit.json]"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from cdsp_inputs import qkv  # noqa: E402
from paper_2511_06247_b200 import api  # noqa: E402

HQ, HKV, D = 32, 8, 128
LS = [4096, 8192, 16384, 32768, 65536]
CS = [0, 16384, 65536, 131072]


def timed(fn, iters):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(iters):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(3_000_000)  # GPU busy while the host enqueues: the events bracket device time
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


def t_s1(C, L, iters, dev):
    plan = api.Plan(([(C, [0])] if C else []) + [(L, [0])])
    c_idx = len(plan.chunks) - 1
    comm = api.Comm(0, 1, 0, api.plan_capacity(plan), HKV, D, torch.bfloat16)
    q, k, v = qkv(C + L, HQ, HKV, D, torch.bfloat16, seed=1, device=dev)
    out = torch.empty(L, HQ, D, dtype=torch.bfloat16, device=dev)
    qc, kc, vc = q[C:].contiguous(), k[C:].contiguous(), v[C:].contiguous()

    def history():
        comm.reset()
        if C:
            api.prefill_chunk(q[:C].contiguous(), k[:C].contiguous(), v[:C].contiguous(), comm.kvstore(),
                              api.SpGroup(comm, plan, 0), 0.0, torch.empty(C, HQ, D, dtype=torch.bfloat16, device=dev))

    ts = []
    for it in range(iters + 2):
        history()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(3_000_000)
        e0.record()
        api.prefill_chunk(qc, kc, vc, comm.kvstore(), api.SpGroup(comm, plan, c_idx), 0.0, out)
        e1.record()
        torch.cuda.synchronize()
        if it >= 2:
            ts.append(e0.elapsed_time(e1))
    comm.close()
    return float(np.median(ts))


def t_ring(s, C, L, iters, dev):
    m = L // (2 * s)
    h = C // s
    q, k, v = qkv(L, HQ, HKV, D, torch.bfloat16, seed=2, device=dev)
    hk = torch.randn(max(h, 1), HKV, D, device=dev).to(torch.bfloat16)[:h]
    shards = []
    for r in range(s):
        ks, vs = api.zigzag_gather(k, s, r), api.zigzag_gather(v, s, r)
        if h:
            ks, vs = torch.cat([hk, ks]).contiguous(), torch.cat([hk, vs]).contiguous()
        shards.append((api.zigzag_gather(q, s, r), ks, vs))
    out = torch.empty(2 * m, HQ, D, dtype=torch.bfloat16, device=dev)
    acc = torch.empty(2 * m, HQ, D, dtype=torch.float32, device=dev)
    lacc = torch.empty(HQ, 2 * m, dtype=torch.float32, device=dev)
    worst = 0.0
    for r in range(s):
        srcs = [(r - st) % s for st in range(s)]
        segs = [api.segments(2 * m, m, C + r * m, C + (2 * s - 1 - r) * m, h + 2 * m, h, m, C + x * m,
                             C + (2 * s - 1 - x) * m) for x in srcs]
        args = (shards[r][0], [shards[x][1] for x in srcs], [shards[x][2] for x in srcs], segs, 0.0, api.ATTN_ONLY)
        worst = max(worst, timed(lambda: api.attention_fwd_blocks(*args, out=out, o_acc=acc, lse_acc=lacc), iters))
    return worst


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=5)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02_eq1_fit.json"))
    ap.add_argument("--sizes", default="1,2,4,8")
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    res = {"what": "Eq. (1) (P:231) fitted on B200 for ONE attention layer, LLaMA3-8B shape (GQA 32/8, d=128, bf16), "
                   "through libcdsp; T in ms",
           "method": {"1": "cdsp_prefill_chunk (chunk after a C-token history chunk), median of CUDA-event timed calls",
                      "s>1": "PROXY: slowest ring rank's fused launch (cdsp_attention_fwd_blocks, peer blocks resident, "
                             "split scratch), ranks timed one at a time on one B200; ring pulls not included"},
           "models": {}, "samples": {}}
    for s in [int(x) for x in a.sizes.split(",")]:
        Cs, Ls, Ts = [], [], []
        for C in CS:
            for L in LS:
                t = t_s1(C, L, a.iters, dev) if s == 1 else t_ring(s, C, L, a.iters, dev)
                Cs.append(C)
                Ls.append(L)
                Ts.append(t)
                print(f"s={s} C={C} L={L}: {t:.3f} ms", flush=True)
        coef = api.fit_latency_model(Cs, Ls, Ts)
        pred = [coef[0] + coef[1] * L + coef[2] * C * L + coef[3] * L * L for C, L in zip(Cs, Ls)]
        rel = [abs(p - t) / t for p, t in zip(pred, Ts)]
        res["models"][str(s)] = {"a": coef[0], "b": coef[1], "c": coef[2], "d": coef[3],
                                 "max_rel_residual": max(rel), "mean_rel_residual": float(np.mean(rel))}
        res["samples"][str(s)] = {"C": Cs, "L": Ls, "T_ms": Ts}
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    with open(a.out, "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps(res["models"], indent=1))


if __name__ == "__main__":
    main()
