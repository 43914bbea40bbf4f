"""Dev: per-CTA timeline of one decode launch (library built with -DCDSP_DTRACE).
Prints quantiles of CTA start / stream-loop end / CTA-merge end / exit relative to the
earliest start (us)."""
import ctypes
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from cdsp_inputs import block_table, qkv  # noqa: E402
from paper_2511_06247_b200 import api  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 262144
Hq, Hkv, D, B, tp = 32, 8, 128, 16, 8
dev = torch.device("cuda:0")
q, k, v = qkv(N, Hq, Hkv, D, torch.bfloat16, seed=0, device=dev)
nl = N // B
bt = block_table(nl, nl + nl // 4, seed=7).to(dev)
kc = [torch.empty((nl + nl // 4, B, 1, D), dtype=torch.bfloat16, device=dev) for _ in range(tp)]
vc = [torch.empty_like(x) for x in kc]
dst = api.DecodeTarget(kc, vc, B, bt)
comm = api.Comm(0, 1, 0, N, Hkv, D, torch.bfloat16)
api.kv_transfer_to_decode(k, v, api.SpGroup(comm, api.Plan([(N, [0])]), 0), dst)
qs = q[N - 1:N, :4].contiguous()
ws = api.decode_workspace(4, 1, D, dev)
L = api.lib()
L.cdsp_debug_decode_trace.argtypes = [ctypes.c_void_p]
buf = np.zeros(4096 * 8, np.uint64)
for it in range(4):
    # flush L2 between runs
    torch.empty(256 << 20, dtype=torch.uint8, device=dev).fill_(1)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    api.decode_attention(qs, dst, 0, 1, N, workspace=ws)
    e1.record()
    torch.cuda.synchronize()
    L.cdsp_debug_decode_trace(buf.ctypes.data)
    t = buf.reshape(4096, 8).astype(np.int64)
    n = int((t[:, 0] > 0).sum())
    t = t[:n]
    t0 = t[:, 0].min()
    rel = (t - t0) / 1e3
    print(f"iter {it}: {n} CTAs, event {e0.elapsed_time(e1) * 1e3:.1f} us")
    for name, col in (("start", 0), ("loop_end", 1), ("merge_end", 2), ("l1_won", 4), ("l1_done", 5),
                      ("l2_won", 6), ("exit", 3)):
        x = rel[:, col][t[:, col] > 0]
        if len(x) == 0:
            continue
        print(f"  {name:9s} n={len(x):4d} q0={np.min(x):7.2f} q10={np.quantile(x, .1):7.2f} q50={np.median(x):7.2f} "
              f"q90={np.quantile(x, .9):7.2f} max={np.max(x):7.2f}")
    sm = t[:, 7] - 1
    le = rel[:, 1]
    by_sm = {}
    for i in range(n):
        by_sm.setdefault(int(sm[i]), []).append(le[i])
    last = np.array([max(v) for v in by_sm.values()])
    print(f"  SMs used {len(by_sm)}; per-SM last loop_end q10={np.quantile(last, .1):.2f} q50={np.median(last):.2f} "
          f"q90={np.quantile(last, .9):.2f}; CTAs/SM {sorted(set(len(v) for v in by_sm.values()))}")
    lo = sorted(by_sm, key=lambda x: max(by_sm[x]))
    print(f"  slowest SMs {lo[-8:]}  fastest SMs {lo[:8]}")
    buf[:] = 0
    torch.cuda.synchronize()
