"""Layer-wise cache-balancing overlap (Fig. 6-b
Fig. 14 "<= 1.8%"): time of the chunk that re-balances history onto a larger group, over
n_layers layers each followed by an FC stand-in (bf16 GEMMs of the model's per-layer FC
FLOPs on the chunk's tokens), in three variants on loopback instances of ONE GPU:
  prebalanced : layer l+1's balancing issued on the comm stream after layer l's ring (default)
  inline      : every layer balances at its own start (CDSP_NO_PREBALANCE=1, in a subprocess)
  control     : the same chunk with history already spread over the group (no balancing)
overhead = (variant - control) / control.  On one GPU the balancing copies run at HBM speed
(not NVLink), so this measures the mechanism's cost; `nvlink_ms_per_layer` projects the
balancing bytes onto a 770 GB/s peer link for context.
usage: python tools/bench_layers.py [--hist 16384] [--chunk 16384] [--layers 8] [--iters 3]"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

import torch  # noqa: E402

from cdsp_inputs import qkv  # noqa: E402
from paper_2511_06247_b200 import api  # noqa: E402
from paper_2511_06247_b200.driver import alloc_out_shards, prepare_shards  # noqa: E402


def run(variant, hist, chunk, n_layers, iters):
    Hq, Hkv, D = 32, 8, 128
    g0 = list(range(4)) if variant != "control" else list(range(8))
    plan_list = [(hist, g0), (chunk, list(range(8)))]
    plan = api.Plan(plan_list)
    N = hist + chunk
    dev = torch.device("cuda:0")
    comms = [api.Comm(i, 8, 0, api.plan_capacity(plan), Hkv, D, torch.bfloat16, n_layers=n_layers) for i in range(8)]
    api.connect_local(comms)
    q, k, v = qkv(N, Hq, Hkv, D, torch.bfloat16, seed=0, device=dev)  # same data for every layer
    shards = prepare_shards(q, k, v, plan)
    outs = alloc_out_shards(plan, Hq, D, torch.bfloat16, dev)
    streams = [torch.cuda.Stream(dev) for _ in range(8)]
    # FC stand-in: LLaMA3-8B per-layer FC FLOPs (QKV 4096x6144, O 4096x4096, MLP 3 x 4096x14336)
    # on this rank's chunk shard of chunk/8 tokens -> one GEMM of equal FLOPs per rank
    tok = chunk // 8
    fc_flops = 2 * tok * 4096 * (6144 + 4096 + 3 * 14336)
    n = int(round((fc_flops / (2 * tok)) ** 0.5 / 128)) * 128
    a = [torch.randn(tok, n, device=dev, dtype=torch.bfloat16) for _ in range(8)]
    w = [torch.randn(n, n, device=dev, dtype=torch.bfloat16) * (1.0 / n ** 0.5) for _ in range(8)]
    cur = torch.cuda.current_stream(dev)

    def chunk_calls(c):
        L, ranks = plan_list[c]
        for l in range(n_layers):
            for r, inst in enumerate(ranks):
                qs, ks, vs = shards[c][r]
                o_r, l_r = outs[c][r]
                api.prefill_chunk(qs, ks, vs, comms[inst].kvstore(l), api.SpGroup(comms[inst], plan, c), 0.0,
                                  o_r, l_r, stream=streams[inst], layer=l)
            if c == 1:
                for r, inst in enumerate(ranks):
                    with torch.cuda.stream(streams[inst]):
                        torch.matmul(a[inst], w[inst])

    times = []
    for it in range(iters + 1):
        for s in streams:
            s.wait_stream(cur)
        for cm in comms:
            cm.reset(cur)
        chunk_calls(0)
        for s in streams:
            cur.wait_stream(s)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(cur)
        for s in streams:
            s.wait_stream(cur)
        chunk_calls(1)
        for s in streams:
            cur.wait_stream(s)
        e1.record(cur)
        torch.cuda.synchronize()
        if it > 0:
            times.append(e0.elapsed_time(e1))
    for cm in comms:
        cm.check()
        cm.close()
    bal_bytes_layer = (hist // 8) * Hkv * D * 2 * 2 * 4  # 4 old ranks each send half of hist/4 tokens
    return {"ms": sorted(times)[len(times) // 2], "fc_tflop_per_layer": 8 * fc_flops / 1e12,
            "balance_bytes_per_layer": bal_bytes_layer}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--hist", type=int, default=16384)
    ap.add_argument("--chunk", type=int, default=16384)
    ap.add_argument("--layers", type=int, default=8)
    ap.add_argument("--iters", type=int, default=3)
    ap.add_argument("--variant", default=None)
    args = ap.parse_args()
    if args.variant:
        print(json.dumps(run(args.variant, args.hist, args.chunk, args.layers, args.iters)))
        return
    res = {}
    for var in ("control", "prebalanced", "inline"):
        env = dict(os.environ)
        if var == "inline":
            env["CDSP_NO_PREBALANCE"] = "1"
        out = subprocess.run([sys.executable, __file__, "--variant", var, "--hist", str(args.hist), "--chunk",
                              str(args.chunk), "--layers", str(args.layers), "--iters", str(args.iters)],
                             capture_output=True, text=True, env=env)
        if out.returncode != 0:
            raise RuntimeError(out.stderr[-2000:])
        res[var] = json.loads(out.stdout.strip().splitlines()[-1])
    ctl = res["control"]["ms"]
    bb = res["prebalanced"]["balance_bytes_per_layer"]
    line = {"metric": "layer-wise cache-balancing overhead (chunk re-balanced 4 -> 8 instances)",
            "hist": args.hist, "chunk": args.chunk, "layers": args.layers, "gpus": 1,
            "ms": {k: v["ms"] for k, v in res.items()},
            "overhead_prebalanced": (res["prebalanced"]["ms"] - ctl) / ctl,
            "overhead_inline": (res["inline"]["ms"] - ctl) / ctl,
            "balance_bytes_per_layer": bb, "nvlink_ms_per_layer_at_770GBps": bb / 4 / 770e9 * 1e3,
            "ms_per_layer_control": ctl / args.layers,
            "note": "8 loopback instances time-share one B200; balancing copies are local (HBM) here"}
    print(json.dumps(line))


if __name__ == "__main__":
    main()
