"""K*1 efficiency, zigzag vs striped: one chunk at SP=s on s loopback
instances of ONE B200 (all ranks' ring steps time-share the GPU, so the chunk's wall time
measures the total attention work as the kernel executes it: masks, partial tiles, skipped
tiles).  TFLOP/s = the chunk's algorithmic FLOPs / wall time.
usage: python tools/bench_interleave.py [--seq 32768] [--heads 32] [--iters 5]"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

import torch  # noqa: E402

from cdsp_inputs import qkv  # noqa: E402
from paper_2511_06247_b200 import api  # noqa: E402
from paper_2511_06247_b200.driver import (alloc_out_shards, make_loopback_comms, prepare_shards,  # noqa: E402
                                          run_plan_loopback)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seq", type=int, default=32768)
    ap.add_argument("--heads", type=int, default=32)
    ap.add_argument("--iters", type=int, default=5)
    ap.add_argument("--zigzag-only", action="store_true")
    ap.add_argument("--one-stream", action="store_true",
                    help="all ranks on one stream: the sum of the ranks' ring times (no time-sharing noise)")
    args = ap.parse_args()
    L, H, D = args.seq, args.heads, 128
    dev = torch.device("cuda:0")
    q, k, v = qkv(L, H, H, D, torch.bfloat16, seed=0, device=dev)
    flops = 4.0 * D * H * L * (L + 1) / 2
    res = {}
    for s in (2, 4, 8):
        for il in (("zigzag",) if args.zigzag_only else ("zigzag", "striped")):
            plan = api.Plan([(L, list(range(s)), il)])
            comms = make_loopback_comms(plan, H, D, torch.bfloat16)
            shards = prepare_shards(q, k, v, plan)
            outs = alloc_out_shards(plan, H, D, torch.bfloat16, dev, want_lse=False)
            one = torch.cuda.Stream(dev)
            streams = [one] * s if args.one_stream else [torch.cuda.Stream(dev) for _ in range(s)]
            times = []
            for it in range(args.iters + 2):
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                run_plan_loopback(q, k, v, plan, comms=comms, streams=streams, want_lse=False, shards=shards,
                                  out_shards=outs)
                e1.record()
                torch.cuda.synchronize()
                if it >= 2:
                    times.append(e0.elapsed_time(e1))
            ms = sorted(times)[len(times) // 2]
            res[f"s{s}_{il}"] = {"ms": ms, "tflops": flops / (ms * 1e-3) / 1e12}
            for c in comms:
                c.close()
    print(json.dumps({"metric": "chunk attention TFLOP/s on one GPU, zigzag vs striped (loopback ranks)",
                      "seq": L, "heads": H, "head_dim": D, "results": res}))


if __name__ == "__main__":
    main()
