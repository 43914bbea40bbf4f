"""HBM-bound kernels of the path, timed alone (CUDA events, median of --iters after warm-up)
against MEASURED_PEAKS.json hbm_gbs; run under ncu (-k regex:<kernel>) for DRAM bytes.
  lse_merge n=2 / n=8 (M2 shape: 32K rows x 32 heads x d=128 fp32 partials -> bf16 out)
  zigzag gather / scatter at s=8 (row_copy_kernel, 32K MHA bf16 q)
  store append (store_append_kernel: k, v shard rows + positions into the store)
  paged scatter (paged_scatter_kernel, M4-like 128K-token shard GQA 8 heads, tp=8)
Algorithmic bytes: merge (n (4D+4) + 2D + 4) B per row-head (bf16 out); row copy 2 x
row bytes per row; append 2 x 2 x row bytes per row + 4 B position; paged 2 x 2 x row bytes per token.
usage: python tools/bench_mem_kernels.py [--iters 20] [--only merge2,merge8,gather,scatter,append,paged]"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from cdsp_inputs import block_table, qkv  # noqa: E402
from paper_2511_06247_b200 import api  # noqa: E402


def timed(fn, iters, per=10):
    """Median over `iters` samples of `per` back-to-back launches (amortises launch latency)."""
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(iters):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(per):
            fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / per)
    return sorted(ts)[len(ts) // 2]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--only", default="merge2,merge8,gather,scatter,append,paged")
    a = ap.parse_args()
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    dev = "cuda"
    res = {}
    T, H, D = 32768, 32, 128
    todo = a.only.split(",")
    for n in (2, 8):
        if f"merge{n}" not in todo:
            continue
        parts = [torch.randn(T, H, D, device=dev) for _ in range(n)]
        lses = [torch.randn(H, T, device=dev) for _ in range(n)]
        out = torch.empty(T, H, D, dtype=torch.bfloat16, device=dev)
        lse = torch.empty(H, T, device=dev)
        ms = timed(lambda: api.lse_merge(parts, lses, out, lse), a.iters)
        by = T * H * (n * (4 * D + 4) + 2 * D + 4)
        res[f"lse_merge_n{n}"] = {"ms": ms, "bytes": by, "gbs": by / ms / 1e6, "frac": by / ms / 1e6 / peak}
        del parts, lses
    q, k, v = qkv(T, H, H, D, torch.bfloat16, seed=0, device=dev)
    s = 8
    shard = torch.empty(T // s, H, D, dtype=torch.bfloat16, device=dev)
    row = H * D * 2
    if "gather" in todo:
        ms = timed(lambda: api.zigzag_gather(q, s, 3, shard), a.iters)
        by = 2 * (T // s) * row
        res["zigzag_gather_s8"] = {"ms": ms, "bytes": by, "gbs": by / ms / 1e6, "frac": by / ms / 1e6 / peak}
    if "scatter" in todo:
        full = torch.empty_like(q)
        ms = timed(lambda: api.zigzag_scatter(shard, s, 3, full), a.iters)
        by = 2 * (T // s) * row
        res["zigzag_scatter_s8"] = {"ms": ms, "bytes": by, "gbs": by / ms / 1e6, "frac": by / ms / 1e6 / peak}
    if "append" in todo:
        # store append inside cdsp_prefill_chunk at s=1 with history: the shard goes through
        # store_append_kernel (k, v rows + positions)
        L = 32768
        plan = api.Plan([(L, [0]), (L, [0])])
        comm = api.Comm(0, 1, 0, api.plan_capacity(plan), H, D, torch.bfloat16)
        ks, vs = k[:L].contiguous(), v[:L].contiguous()
        qs = q[:64].contiguous()  # queries do not matter here; the append is timed via ncu

        def app():
            comm.reset()
            api.prefill_chunk(q[:L], ks, vs, comm.kvstore(), api.SpGroup(comm, plan, 0))
            api.prefill_chunk(q[:L], ks, vs, comm.kvstore(), api.SpGroup(comm, plan, 1))
        app()
        torch.cuda.synchronize()
        res["store_append"] = {"note": "append of chunk 1 (32K rows, history 32K) inside cdsp_prefill_chunk; "
                                       "time it from the ncu launch list (store_append_kernel)",
                               "bytes": 2 * 2 * L * row + 4 * L}
        del qs
        comm.close()
    if "paged" in todo:
        N, Hkv, tp, B = 131072, 8, 8, 16
        kk = torch.randn(N, Hkv, D, device=dev).to(torch.bfloat16)
        vv = torch.randn(N, Hkv, D, device=dev).to(torch.bfloat16)
        nl = N // B
        bt = block_table(nl, nl + 1024, seed=7).to(dev)
        kc = [torch.empty(nl + 1024, B, Hkv // tp, D, dtype=torch.bfloat16, device=dev) for _ in range(tp)]
        vc = [torch.empty_like(x) for x in kc]
        dst = api.DecodeTarget(kc, vc, B, bt)
        plan = api.Plan([(N, [0])])
        comm = api.Comm(0, 1, 0, N, Hkv, D, torch.bfloat16)
        g = api.SpGroup(comm, plan, 0)
        ms = timed(lambda: api.kv_transfer_to_decode(kk, vv, g, dst), a.iters)
        by = 2 * 2 * N * Hkv * D * 2
        res["paged_scatter_128k_gqa"] = {"ms": ms, "bytes": by, "gbs": by / ms / 1e6, "frac": by / ms / 1e6 / peak}
        comm.close()
    print(json.dumps({"peak_hbm_gbs": peak, "results": res}, indent=1))


if __name__ == "__main__":
    main()
