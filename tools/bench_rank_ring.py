"""Per-GPU ring compute at SP = s, on one B200: the attention ONE rank of an s-GPU ring runs
for a chunk, with the peer blocks already resident (the ring pulls run on copy engines and
are timed by bench.py's `ring` field on a real multi-GPU run).  Two designs:
  split:    one cdsp_attention_fwd_blocks launch walking all s blocks (step 0 self/causal,
            then src = (r - k) mod s, P:59 / R10-R11) with O resident in TMEM, heavy units split
            over two block ranges and merged through the accumulator scratch — what
            cdsp_prefill_chunk runs when accumulators are reserved;
  fused:    the same without scratch (no splitting);
  stepwise: s cdsp_attention_fwd launches FIRST / MID / LAST merged through fp32
            accumulators (MID / LAST as programmatic dependents) — the round-1 design.
Every rank r = 0..s-1 is timed on its own, back to back on one stream; a real ring ends when
its slowest rank does, so the per-GPU rate is chunk FLOPs / s / max_r(time_r).  Zigzag shards
(P:75); optional history (--hist-per-rank rows of earlier chunks on every rank, always visible).
usage: python tools/bench_rank_ring.py [--seq 32768] [--heads 32] [--kv-heads 32] [--iters 10]
       [--sizes 1,2,4,8] [--hist-per-rank 0] [--modes fused,stepwise]"""
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
    ap.add_argument("--kv-heads", type=int, default=None)
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--per", type=int, default=1, help="back-to-back rank runs per timed sample")
    ap.add_argument("--sizes", default="1,2,4,8")
    ap.add_argument("--hist-per-rank", type=int, default=0)
    ap.add_argument("--modes", default="split,fused,stepwise")
    ap.add_argument("--ranks", default="all", help="'all' or a comma list of ring ranks to time")
    args = ap.parse_args()
    L, H, D = args.seq, args.heads, 128
    Hkv = args.kv_heads or H
    h = args.hist_per_rank
    dev = torch.device("cuda:0")
    q, k, v = qkv(L, H, Hkv, D, torch.bfloat16, seed=0, device=dev)
    res = {}
    for s in [int(x) for x in args.sizes.split(",")]:
        m = L // (2 * s)
        C = s * h
        # block of src: h history rows (random keys: values do not matter for timing) + its shard
        hk = torch.randn(h, Hkv, D, device=dev).to(torch.bfloat16) if h else None
        shards = []
        for r in range(s):
            qs, ks, vs = api.zigzag_gather(q, s, r), api.zigzag_gather(k, s, r), api.zigzag_gather(v, s, r)
            if h:
                ks, vs = torch.cat([hk, ks]).contiguous(), torch.cat([hk, vs]).contiguous()
            shards.append((qs, ks, vs))
        o_acc = torch.empty(2 * m, H, D, dtype=torch.float32, device=dev)
        lse_acc = torch.empty(H, 2 * m, dtype=torch.float32, device=dev)
        out = torch.empty(2 * m, H, D, dtype=torch.bfloat16, device=dev)

        def pos0(r):
            return C + r * m

        def pos1(r):
            return C + (2 * s - 1 - r) * m

        def seg(r, src):
            return api.segments(2 * m, m, pos0(r), pos1(r), h + 2 * m, h, m, pos0(src), pos1(src))

        def run_rank(r, mode):
            if mode in ("fused", "split") or s == 1:
                srcs = [(r - step) % s for step in range(s)]
                scratch = dict(o_acc=o_acc, lse_acc=lse_acc) if mode == "split" else {}
                api.attention_fwd_blocks(shards[r][0], [shards[x][1] for x in srcs], [shards[x][2] for x in srcs],
                                         [seg(r, x) for x in srcs], 0.0, api.ATTN_ONLY, out=out, **scratch)
                return
            for step in range(s):
                src = (r - step) % s
                md = api.ATTN_FIRST if step == 0 else (api.ATTN_LAST if step == s - 1 else api.ATTN_MID) | api.ATTN_PDL
                _, ks, vs = shards[src]
                api.attention_fwd(shards[r][0], ks, vs, seg(r, src), 0.0, md, o_acc=o_acc, lse_acc=lse_acc, out=out)

        ranks = range(s) if args.ranks == "all" else [int(x) for x in args.ranks.split(",") if int(x) < s]
        for mode in args.modes.split(","):
            if s == 1 and mode != args.modes.split(",")[0]:
                continue
            per_rank = []
            for r in ranks:
                for _ in range(2):
                    run_rank(r, mode)
                torch.cuda.synchronize()
                ts = []
                for _ in range(args.iters):  # `per` back-to-back rank runs per sample
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    torch.cuda._sleep(3_000_000)  # GPU busy while the host marshals and enqueues: device time only
                    e0.record()
                    for _ in range(args.per):
                        run_rank(r, mode)
                    e1.record()
                    torch.cuda.synchronize()
                    ts.append(e0.elapsed_time(e1) / args.per)
                per_rank.append(sorted(ts)[len(ts) // 2])
            flops = 4.0 * D * H * (L * C + L * (L + 1) / 2)
            tmax = max(per_rank)
            res[f"s{s}_{mode if s > 1 else 'single'}"] = {
                "rank_ms_max": tmax, "rank_ms_min": min(per_rank), "ranks_timed": len(per_rank),
                "rank_ms": [round(x, 4) for x in per_rank],
                "tflops_per_gpu": flops / s / (tmax * 1e-3) / 1e12}
    print(json.dumps({"metric": "per-GPU ring attention TFLOP/s at SP=s (one rank's launches, peer blocks resident)",
                      "seq": L, "heads": H, "kv_heads": Hkv, "head_dim": D, "hist_per_rank": h, "results": res}))


if __name__ == "__main__":
    main()
