"""Dev: per-CTA timeline of one batched decode launch (library built with -DCDSP_DTRACE):
quantiles of CTA start / stream-loop end / exit (us from the earliest start) and the stream
time per 64-token stage, for equal vs mixed lengths.
usage: python tools/decode_batch_trace.py [--batch 32] [--ctx 32768] [--mixed]"""
import argparse
import ctypes
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2511_06247_b200 import api  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=32)
ap.add_argument("--ctx", type=int, default=32768)
ap.add_argument("--mixed", action="store_true")
a = ap.parse_args()
B, D, hq_t, hkv_t, tp = 16, 128, 4, 1, 1
dev = torch.device("cuda:0")
g = torch.Generator().manual_seed(11)
lens = (torch.randint(a.ctx // 4, a.ctx + 1, (a.batch,), generator=g) if a.mixed
        else torch.full((a.batch,), a.ctx, dtype=torch.int64))
pages = (lens + B - 1) // B
pool = int(pages.sum()) + 64
perm = torch.randperm(pool, generator=g).to(torch.int32)
bt = torch.full((a.batch, int(pages.max())), -1, dtype=torch.int32)
o = 0
for b in range(a.batch):
    n = int(pages[b])
    bt[b, :n] = perm[o:o + n]
    o += n
gd = torch.Generator(device=dev).manual_seed(5)
kc = [torch.randn((pool, B, hkv_t, D), generator=gd, device=dev).to(torch.bfloat16)]
vc = [torch.randn((pool, B, hkv_t, D), generator=gd, device=dev).to(torch.bfloat16)]
dst = api.DecodeTarget(kc, vc, B, bt.to(dev))
q = torch.randn((a.batch, hq_t, D), generator=gd, device=dev).to(torch.bfloat16)
ws = api.decode_workspace(a.batch * hq_t, a.batch * hkv_t, D, dev)
L = api.lib()
L.cdsp_debug_decode_trace.argtypes = [ctypes.c_void_p]
buf = np.zeros(4096 * 8, np.uint64)
lh = [int(x) for x in lens]
for it in range(3):
    torch.empty(256 << 20, dtype=torch.uint8, device=dev).fill_(1)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    api.decode_attention_batch(q, dst, 0, hkv_t, lh, workspace=ws)
    e1.record()
    torch.cuda.synchronize()
    L.cdsp_debug_decode_trace(buf.ctypes.data)
    t = buf.reshape(4096, 8).astype(np.int64)
    n = int((t[:, 0] > 0).sum())
    t = t[:n]
    rel = (t - t[:, 0].min()) / 1e3
    print(f"iter {it}: {n} CTAs, event {e0.elapsed_time(e1) * 1e3:.1f} us, SMs {len(set((t[:, 7] - 1).tolist()))}")
    for name, col in (("start", 0), ("loop_end", 1), ("merge_end", 2), ("exit", 3)):
        x = rel[:, col][t[:, col] > 0]
        print(f"  {name:9s} q0={np.min(x):7.2f} q10={np.quantile(x, .1):7.2f} q50={np.median(x):7.2f} "
              f"q90={np.quantile(x, .9):7.2f} max={np.max(x):7.2f}")
    dur = rel[:, 1] - rel[:, 0]
    print(f"  stream (loop_end - start) q10={np.quantile(dur, .1):.2f} q50={np.median(dur):.2f} max={dur.max():.2f} us")
    per_sm = {}
    for i in range(n):
        per_sm.setdefault(int(t[i, 7]), 0)
        per_sm[int(t[i, 7])] += 1
    c = np.bincount(list(per_sm.values()))
    print(f"  CTAs per SM histogram: {dict(enumerate(c.tolist()))}")
