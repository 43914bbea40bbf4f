"""Per-GPU ring compute at SP = s, on one B200: the s block-attention launches ONE rank of an
s-GPU ring issues for a chunk (step 0 self/causal, FIRST; steps 1..s-1 the blocks of
src = (r - k) mod s, MID, the last one LAST, P:59 / R10-R11), with the peer blocks already
resident (the ring pulls run on copy engines and are timed separately by bench.py's `ring`
field on a real multi-GPU run).  Every rank r = 0..s-1 is timed on its own, back to back on
one stream; a real ring step ends when its slowest rank does, so the per-GPU rate is
chunk FLOPs / s / max_r(time_r).  Zigzag shards.
usage: python tools/bench_rank_ring.py [--seq 32768] [--heads 32] [--iters 10]"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from cdsp_inputs import qkv  # noqa: E402
from paper_2511_06247_b200 import api  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seq", type=int, default=32768)
    ap.add_argument("--heads", type=int, default=32)
    ap.add_argument("--iters", type=int, default=10)
    args = ap.parse_args()
    L, H, D = args.seq, args.heads, 128
    dev = torch.device("cuda:0")
    q, k, v = qkv(L, H, H, D, torch.bfloat16, seed=0, device=dev)
    res = {}
    for s in (1, 2, 4, 8):
        m = L // (2 * s)
        shards = [(api.zigzag_gather(q, s, r), api.zigzag_gather(k, s, r), api.zigzag_gather(v, s, r))
                  for r in range(s)]
        o_acc = torch.empty(2 * m, H, D, dtype=torch.float32, device=dev)
        lse_acc = torch.empty(H, 2 * m, dtype=torch.float32, device=dev)
        out = torch.empty(2 * m, H, D, dtype=torch.bfloat16, device=dev)

        def pos0(r):
            return r * m

        def pos1(r):
            return (2 * s - 1 - r) * m

        def run_rank(r):
            for step in range(s):
                src = (r - step) % s
                seg = api.segments(2 * m, m, pos0(r), pos1(r), 2 * m, 0, m, pos0(src), pos1(src))
                mode = (api.ATTN_ONLY if s == 1 else
                        api.ATTN_FIRST if step == 0 else api.ATTN_LAST if step == s - 1 else api.ATTN_MID)
                _, ks, vs = shards[src]
                api.attention_fwd(shards[r][0], ks, vs, seg, 0.0, mode, o_acc=o_acc, lse_acc=lse_acc, out=out)

        per_rank = []
        for r in range(s):
            for _ in range(2):
                run_rank(r)
            torch.cuda.synchronize()
            ts = []
            for _ in range(args.iters):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                run_rank(r)
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            per_rank.append(sorted(ts)[len(ts) // 2])
        flops = 4.0 * D * H * L * (L + 1) / 2
        tmax = max(per_rank)
        res[f"s{s}"] = {"rank_ms_max": tmax, "rank_ms_min": min(per_rank),
                        "tflops_per_gpu": flops / s / (tmax * 1e-3) / 1e12}
    print(json.dumps({"metric": "per-GPU ring attention TFLOP/s at SP=s (one rank's s launches, peer blocks resident)",
                      "seq": L, "heads": H, "head_dim": D, "results": res}))


if __name__ == "__main__":
    main()
