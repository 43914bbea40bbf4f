"""One fused ring launch of ring rank r at SP = s (peer blocks resident) for ncu:
launch 0 warms up, launch 1 is the one to capture (ncu -k regex:attn_tc -s 1 -c 1).
usage: python tools/ncu_fused_rank.py --s 8 --r 0 [--seq 32768 --heads 32 --kv-heads 32]"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from cdsp_inputs import qkv  # noqa: E402
from paper_2511_06247_b200 import api  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--s", type=int, default=8)
ap.add_argument("--r", type=int, default=0)
ap.add_argument("--seq", type=int, default=32768)
ap.add_argument("--heads", type=int, default=32)
ap.add_argument("--kv-heads", type=int, default=None)
ap.add_argument("--launches", type=int, default=2)
ap.add_argument("--split", action="store_true", help="pass accumulator scratch (heavy units split)")
a = ap.parse_args()
L, H, D, s, r = a.seq, a.heads, 128, a.s, a.r
Hkv = a.kv_heads or H
q, k, v = qkv(L, H, Hkv, D, torch.bfloat16, seed=0, device="cuda")
m = L // (2 * s)
sh = [(api.zigzag_gather(q, s, x), api.zigzag_gather(k, s, x), api.zigzag_gather(v, s, x)) for x in range(s)]
srcs = [(r - step) % s for step in range(s)]
segs = [api.segments(2 * m, m, r * m, (2 * s - 1 - r) * m, 2 * m, 0, m, x * m, (2 * s - 1 - x) * m) for x in srcs]
out = torch.empty_like(sh[r][0])
kw = {}
if a.split:
    kw = dict(o_acc=torch.empty(2 * m, H, D, dtype=torch.float32, device="cuda"),
              lse_acc=torch.empty(H, 2 * m, dtype=torch.float32, device="cuda"))
for _ in range(a.launches):
    api.attention_fwd_blocks(sh[r][0], [sh[x][1] for x in srcs], [sh[x][2] for x in srcs], segs, 0.0, api.ATTN_ONLY,
                             out=out, **kw)
torch.cuda.synchronize()
print("flops", 4.0 * D * H * L * (L + 1) / 2 / s)
