"""Dev: is the s=1 kernel's run-to-run spread (two modes, ~1360 vs ~1410 TF/s) a property of the
process (allocation addresses) or of the launch?  Times 12 launches of the 32K MHA chunk for
several allocation offsets (a pad tensor before q/k/v) in one process."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from cdsp_inputs import qkv  # noqa: E402
from paper_2511_06247_b200 import api  # noqa: E402

L, H, D = 32768, 32, 128
dev = torch.device("cuda:0")
flops = 4.0 * D * H * L * (L + 1) / 2
q0, k0, v0 = qkv(L, H, H, D, torch.bfloat16, seed=0, device=dev)
seg = api.causal_segments(L, L)
for pad_mb in [0, 1, 2, 3, 5, 8, 13, 21, 34]:
    pad = torch.empty(pad_mb << 20, dtype=torch.uint8, device=dev) if pad_mb else None
    q, k, v = q0.clone(), k0.clone(), v0.clone()
    out = torch.empty_like(q)
    ts = []
    for it in range(14):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(2_000_000)
        e0.record()
        api.attention_fwd(q, k, v, seg, 0.0, api.ATTN_ONLY, out=out)
        e1.record()
        torch.cuda.synchronize()
        if it >= 2:
            ts.append(e0.elapsed_time(e1))
    tf = [flops / (t * 1e-3) / 1e12 for t in ts]
    print(f"pad {pad_mb:3d} MB q@{q.data_ptr() % (1 << 30):#x}: TF/s " + " ".join(f"{x:.0f}" for x in tf), flush=True)
    del q, k, v, out, pad
    torch.cuda.empty_cache()
