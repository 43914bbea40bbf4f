"""Per-GPU chunk latency of whole CDSP plans on one B200 (compute side of the ring).

For every chunk c of a plan (chunk c runs on s_c instances, its history C_c evenly
re-balanced onto them, R8) and every ring rank r of its group, the s_c block-attention launches
rank r issues (step k: Q = r's zigzag shard, KV = src's C_c/s_c history rows + src's shard,
src = (r - k) mod s_c; FIRST / MID / LAST, fused LSE merge) are timed back to back on one stream
with the peer blocks resident (the pulls run on copy engines; a real ring hides them when the
chunk's compute/comm ratio is high).  Chunk latency = the slowest rank; TFLOP/s per
GPU = chunk FLOPs / s_c / latency.  History rows carry no positions (always visible), so
the KV contents are synthetic; timing only.
usage: python tools/bench_plan_rank.py [--configs M3 M4 M5] [--iters 3]"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2511_06247_b200 import api  # noqa: E402

K = 1024
PLANS = {  # name: (chunks [(len, s)], Hq, Hkv) -- SURVEY 8(d) M3 plan A, M4, M5 (s = 8)
    "M3": ([(32 * K, 2), (32 * K, 4), (32 * K, 8), (32 * K, 8)], 32, 32),
    "M4": ([(64 * K, 2), (64 * K, 4), (128 * K, 8)], 32, 8),
    "M5": ([(512 * K, 8)], 32, 8),
}


def chunk_latency(L, s, C, Hq, Hkv, iters, dev):
    D = 128
    m = L // (2 * s)
    h = C // s
    g = torch.Generator(device=dev).manual_seed(7)
    q = torch.randn(2 * m, Hq, D, generator=g, device=dev).to(torch.bfloat16)
    kv = [torch.randn(h + 2 * m, Hkv, D, generator=g, device=dev).to(torch.bfloat16) for _ in range(2)]
    o_acc = torch.empty(2 * m, Hq, D, dtype=torch.float32, device=dev)
    lse_acc = torch.empty(Hq, 2 * m, dtype=torch.float32, device=dev)
    out = torch.empty(2 * m, Hq, D, dtype=torch.bfloat16, device=dev)

    def p0(x):
        return C + x * m

    def p1(x):
        return C + (2 * s - 1 - x) * m

    def run_rank(r):
        for step in range(s):
            src = (r - step) % s
            seg = api.segments(2 * m, m, p0(r), p1(r), h + 2 * m, h, m, p0(src), p1(src))
            mode = (api.ATTN_ONLY if s == 1 else api.ATTN_FIRST if step == 0 else
                    api.ATTN_LAST if step == s - 1 else api.ATTN_MID)
            api.attention_fwd(q, kv[0], kv[1], seg, 0.0, mode, o_acc=o_acc, lse_acc=lse_acc, out=out)

    times = []
    for r in range(s):
        run_rank(r)
        torch.cuda.synchronize()
        ts = []
        for _ in range(iters):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            run_rank(r)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        times.append(sorted(ts)[len(ts) // 2])
    flops = 4.0 * D * Hq * (L * C + L * (L + 1) / 2)
    lat = max(times)
    return {"L": L, "s": s, "history": C, "latency_ms": lat, "rank_ms_min": min(times),
            "tflops_per_gpu": flops / s / (lat * 1e-3) / 1e12}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", nargs="*", default=["M3", "M4", "M5"])
    ap.add_argument("--iters", type=int, default=3)
    args = ap.parse_args()
    dev = torch.device("cuda:0")
    res = {}
    for name in args.configs:
        chunks, Hq, Hkv = PLANS[name]
        C = 0
        rows = []
        for L, s in chunks:
            rows.append(chunk_latency(L, s, C, Hq, Hkv, args.iters, dev))
            C += L
        res[name] = {"q_heads": Hq, "kv_heads": Hkv, "chunks": rows,
                     "prefill_latency_ms": sum(x["latency_ms"] for x in rows)}
    print(json.dumps({"metric": "per-GPU chunk latency of CDSP plans (one rank's launches, peer blocks resident)",
                      "results": res}))


if __name__ == "__main__":
    main()
