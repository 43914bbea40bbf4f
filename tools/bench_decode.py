"""Decode-consumer bench: cdsp_decode_attention over the paged caches
cdsp_kv_transfer_to_decode writes, LLaMA3-8B GQA shape (32 Q / 8 KV heads, d=128, bf16),
decode tp=8 (1 KV head, 4 Q heads per rank), block 16, seeded block table.

One "step" = the decode attention of all 8 decode TP ranks for one new token (on one GPU the
8 ranks' launches run back to back; each rank's cache is 134 MB at 256K, 1.07 GB in total,
so every launch streams from HBM: the 126 MB L2 holds at most one rank's cache and each is
revisited 8 launches later).  Per-launch times by CUDA event pairs on the launching stream.
Roofline: HBM; algorithmic bytes per launch = n_ctx x Hkv_t x D x 2 (K, V) x 2 B + block
table (4 B per block) + q/out; peak = MEASURED_PEAKS.json hbm_gbs.
usage: python tools/bench_decode.py [--ctx 262144] [--steps 20] [--warmup 3]"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from cdsp_inputs import block_table, qkv  # noqa: E402
from paper_2511_06247_b200 import api  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ctx", type=int, default=262144)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--tp", type=int, default=8)
    ap.add_argument("--identity-table", action="store_true", help="block table = 0, 1, 2, ... (dev)")
    args = ap.parse_args()
    Hq, Hkv, D, B, tp = 32, 8, 128, 16, args.tp
    N = args.ctx
    dev = torch.device("cuda:0")
    q, k, v = qkv(N, Hq, Hkv, D, torch.bfloat16, seed=0, device=dev)
    n_logical = N // B
    nb = n_logical + n_logical // 4
    bt = block_table(n_logical, nb, seed=7).to(dev)
    if args.identity_table:
        bt = torch.arange(n_logical, dtype=torch.int32, device=dev)
    kc = [torch.empty((nb, B, Hkv // tp, D), dtype=torch.bfloat16, device=dev) for _ in range(tp)]
    vc = [torch.empty_like(x) for x in kc]
    dst = api.DecodeTarget(kc, vc, B, bt)
    comm = api.Comm(0, 1, 0, N, Hkv, D, torch.bfloat16)
    api.kv_transfer_to_decode(k, v, api.SpGroup(comm, api.Plan([(N, [0])]), 0), dst)
    del k, v
    hq_t, hkv_t = Hq // tp, Hkv // tp
    qs = [q[N - 1:N, t * hq_t:(t + 1) * hq_t].contiguous() for t in range(tp)]
    outs = [torch.empty_like(x) for x in qs]
    lses = [torch.empty(hq_t, dtype=torch.float32, device=dev) for _ in range(tp)]
    wss = [api.decode_workspace(hq_t, hkv_t, D, dev) for _ in range(tp)]
    st = torch.cuda.current_stream(dev)

    def step(evs=None):
        for t in range(tp):
            if evs is not None:
                evs[t][0].record(st)
            api.decode_attention(qs[t], dst, t, hkv_t, N, out=outs[t], lse=lses[t], workspace=wss[t], stream=st)
            if evs is not None:
                evs[t][1].record(st)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    evs = [[[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(tp)] for _ in range(args.steps)]
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for i in range(args.steps):
        step(evs[i])
    e1.record(st)
    torch.cuda.synchronize()
    launch_ms = [evs[i][t][0].elapsed_time(evs[i][t][1]) for i in range(args.steps) for t in range(tp)]
    avg = sum(launch_ms) / len(launch_ms)
    bytes_launch = N * hkv_t * D * 2 * 2 + (N // B) * 4 + 2 * hq_t * D * 2 + hq_t * 4
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    gbs = bytes_launch / (avg * 1e-3) / 1e9
    line = {"metric": "decode attention over the transferred paged cache (GB/s)", "value": gbs, "unit": "GB/s",
            "ctx": N, "tp": tp, "q_heads": Hq, "kv_heads": Hkv, "head_dim": D, "block": B, "dtype": "bf16",
            "avg_launch_us": avg * 1e3, "min_launch_us": min(launch_ms) * 1e3,
            "step_us_all_ranks": e0.elapsed_time(e1) / args.steps * 1e3, "launches": len(launch_ms),
            "roofline": {"bound": "hbm", "achieved": gbs, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                         "frac": gbs / peaks["hbm_gbs"], "bytes_per_launch": bytes_launch}}
    print(json.dumps(line), flush=True)
    comm.close()


if __name__ == "__main__":
    main()
