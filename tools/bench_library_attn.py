"""Context numbers (not the product, not the target): the installed libraries' causal prefill
attention on the bench's s = 1 workload (32K MHA 32/32, d = 128, bf16), same box, CUDA events.

    python tools/bench_library_attn.py --backend {cudnn,flash2,fi_fa2,ours}

One JSON line per call: TFLOP/s = 4·d·Hq·L(L+1)/2 (the visible causal pairs, the same count
bench.py uses) / average launch time over `--iters` back-to-back launches after warm-up.  Run each
backend in its own process (a failing JIT or a missing cubin must not take the others down)."""
import argparse
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402


def timed(fn, iters, warm):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    time.sleep(0.3)  # same idle gap as bench.py before its timed region
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--backend", required=True)
    ap.add_argument("--L", type=int, default=32768)
    ap.add_argument("--hq", type=int, default=32)
    ap.add_argument("--hkv", type=int, default=32)
    ap.add_argument("--d", type=int, default=128)
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--warm", type=int, default=3)
    a = ap.parse_args()
    L, Hq, Hkv, D = a.L, a.hq, a.hkv, a.d
    dev = torch.device("cuda:0")
    g = torch.Generator(device=dev).manual_seed(0)
    q = torch.randn(L, Hq, D, device=dev, dtype=torch.bfloat16, generator=g)
    k = torch.randn(L, Hkv, D, device=dev, dtype=torch.bfloat16, generator=g)
    v = torch.randn(L, Hkv, D, device=dev, dtype=torch.bfloat16, generator=g)
    scale = 1.0 / math.sqrt(D)
    flops = 4.0 * D * Hq * (L * (L + 1) / 2)
    b = a.backend
    note = ""
    if b in ("cudnn", "flash2"):
        from torch.nn.attention import SDPBackend, sdpa_kernel
        import torch.nn.functional as F
        qt, kt, vt = (x.transpose(0, 1).unsqueeze(0) for x in (q, k, v))  # [1, H, L, D] views
        be = SDPBackend.CUDNN_ATTENTION if b == "cudnn" else SDPBackend.FLASH_ATTENTION
        note = f"torch {torch.__version__} SDPA {be.name}, [1,H,L,D] strided views of NHD"

        def fn():
            with sdpa_kernel([be]):
                return F.scaled_dot_product_attention(qt, kt, vt, is_causal=True, scale=scale,
                                                      enable_gqa=Hq != Hkv)
    elif b.startswith("fi_"):
        import flashinfer
        be = {"fi_fa2": "fa2"}[b]  # (the installed flashinfer's single-prefill API offers fa2 / fa3 only)
        note = f"flashinfer {flashinfer.__version__} single_prefill_with_kv_cache backend={be}"

        def fn():
            return flashinfer.single_prefill_with_kv_cache(q, k, v, causal=True, sm_scale=scale,
                                                           backend=be)
    elif b == "ours":
        from paper_2511_06247_b200 import api
        out = torch.empty_like(q)
        lse = torch.empty(Hq, L, device=dev, dtype=torch.float32)
        note = "cdsp_attention_fwd (ONLY mode, s = 1 causal)"
        seg = api.causal_segments(L, L)

        def fn():
            api.attention_fwd(q, k, v, seg, scale, api.ATTN_ONLY, out=out, lse=lse)
    else:
        raise SystemExit(f"unknown backend {b}")
    try:
        ms = timed(fn, a.iters, a.warm)
        rec = {"backend": b, "L": L, "hq": Hq, "hkv": Hkv, "d": D, "ms": ms,
               "tflops": flops / ms / 1e9, "iters": a.iters, "note": note,
               "gpu": torch.cuda.get_device_name(0)}
    except Exception as e:  # noqa: BLE001 - context tool: report, do not crash the sweep
        rec = {"backend": b, "error": f"{type(e).__name__}: {str(e)[:300]}", "note": note}
    print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()
