"""Batched decode bench (widened to a decode instance's batch):
cdsp_decode_attention_batch on decode TP rank 0, LLaMA3-8B GQA shape (32 Q / 8 KV heads, d=128,
bf16), tp=8 (1 KV head, 4 Q heads per rank), block 16, every request's pages a seeded random
slice of one shared pool (as a paged allocator hands them out).  Context lengths: `--ctx` each,
or a seeded mix in [ctx/4, ctx] with `--mixed`.

One launch per step (all requests).  Per-launch time by CUDA event pairs on the launching stream,
after warm-up; the pool (batch x ctx x 512 B) exceeds the 126 MB L2 for batch x ctx >= 256K, and
consecutive launches read it in the same order, so the L2 holds at most its tail.
Roofline: HBM; algorithmic bytes per launch = sum_b ctx_b x Hkv_t x D x 2 (K, V) x 2 B + block
table rows + q / out; peak = MEASURED_PEAKS.json hbm_gbs.
usage: python tools/bench_decode_batch.py [--batch 16] [--ctx 32768] [--mixed] [--steps 20]"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2511_06247_b200 import api  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=16)
    ap.add_argument("--ctx", type=int, default=32768)
    ap.add_argument("--mixed", action="store_true")
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    args = ap.parse_args()
    Hq, Hkv, D, B, tp = 32, 8, 128, 16, 8
    hq_t, hkv_t = Hq // tp, Hkv // tp
    nb_req = args.batch
    dev = torch.device("cuda:0")
    g = torch.Generator().manual_seed(11)
    if args.mixed:
        lens = torch.randint(args.ctx // 4, args.ctx + 1, (nb_req,), generator=g)
    else:
        lens = torch.full((nb_req,), args.ctx, dtype=torch.int64)
    pages = (lens + B - 1) // B
    row = int(pages.max())
    pool = int(pages.sum()) + 64
    perm = torch.randperm(pool, generator=g).to(torch.int32)
    bt = torch.full((nb_req, row), -1, dtype=torch.int32)
    o = 0
    for b in range(nb_req):
        n = int(pages[b])
        bt[b, :n] = perm[o:o + n]
        o += n
    bt = bt.to(dev)
    # the cache contents do not change the traffic: seeded random bf16 (rank 0's one KV head)
    gd = torch.Generator(device=dev).manual_seed(5)
    kc = [torch.randn((pool, B, hkv_t, D), generator=gd, device=dev).to(torch.bfloat16) for _ in range(tp)]
    vc = [torch.randn((pool, B, hkv_t, D), generator=gd, device=dev).to(torch.bfloat16) for _ in range(tp)]
    dst = api.DecodeTarget(kc, vc, B, bt)
    q = torch.randn((nb_req, hq_t, D), generator=gd, device=dev).to(torch.bfloat16)
    out = torch.empty_like(q)
    lse = torch.empty((nb_req, hq_t), dtype=torch.float32, device=dev)
    lens_h = [int(x) for x in lens]
    tot = int(lens.sum())
    ws = api.decode_workspace(nb_req * hq_t, nb_req * hkv_t, D, dev)
    st = torch.cuda.current_stream(dev)

    def step():
        api.decode_attention_batch(q, dst, 0, hkv_t, lens_h, out=out, lse=lse, workspace=ws, stream=st)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(args.steps)]
    for i in range(args.steps):
        evs[i][0].record(st)
        step()
        evs[i][1].record(st)
    torch.cuda.synchronize()
    ms = [a.elapsed_time(b) for a, b in evs]
    avg = sum(ms) / len(ms)
    bytes_launch = tot * hkv_t * D * 2 * 2 + int(pages.sum()) * 4 + nb_req * (2 * hq_t * D * 2 + hq_t * 4)
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    gbs = bytes_launch / (avg * 1e-3) / 1e9
    line = {"metric": "batched decode attention over paged caches (GB/s)", "value": gbs, "unit": "GB/s",
            "batch": nb_req, "ctx": args.ctx, "mixed": args.mixed, "tokens": tot, "tp": tp, "rank": 0,
            "q_heads": Hq, "kv_heads": Hkv, "head_dim": D, "block": B, "dtype": "bf16",
            "avg_launch_us": avg * 1e3, "min_launch_us": min(ms) * 1e3, "bytes_per_launch": bytes_launch,
            "hbm_peak_gbs": peaks["hbm_gbs"], "frac_of_hbm": gbs / peaks["hbm_gbs"], "steps": args.steps,
            "timing": "CUDA events around each launch, after warm-up"}
    print(json.dumps(line))


if __name__ == "__main__":
    main()
