"""Dev: CTA timelines (build with CDSP_KTRACE=1) of (a) the s=1 32K causal launch and (b) one
SP=8 ring step of the 32K chunk (rank 3 attending src 1's shard, MID merge mode), to size the
per-CTA fixed cost against the per-tile work."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

import torch  # noqa: E402

from cdsp_inputs import qkv  # noqa: E402
from paper_2511_06247_b200 import api  # noqa: E402
from trace_attn import analyze_ctas  # noqa: E402

out_dir = sys.argv[1]
H, D = 32, 128
# (a) s = 1
N = 32768
q, k, v = qkv(N, H, H, D, torch.bfloat16, seed=0, device="cuda")
out = torch.empty_like(q)
api.attention_fwd(q, k, v, api.causal_segments(N, N), 0.0, api.ATTN_ONLY, out=out)
torch.cuda.synchronize()
os.environ["CDSP_TRACE"] = os.path.join(out_dir, "trace_s1.bin")
api.attention_fwd(q, k, v, api.causal_segments(N, N), 0.0, api.ATTN_ONLY, out=out)
torch.cuda.synchronize()
del os.environ["CDSP_TRACE"]
print("== s=1 32K causal")
analyze_ctas(os.path.join(out_dir, "trace_s1.bin"), 8192)
# (b) ring step s=8, r=3, src=1 (src < r: all q x first half of the src shard)
s, m = 8, N // 16
qs, ks, vs = q[: 2 * m].contiguous(), k[: 2 * m].contiguous(), v[: 2 * m].contiguous()
r, src = 3, 1
seg = api.segments(2 * m, m, r * m, (2 * s - 1 - r) * m, 2 * m, 0, m, src * m, (2 * s - 1 - src) * m)
o_acc = torch.zeros(2 * m, H, D, dtype=torch.float32, device="cuda")
lse_acc = torch.zeros(H, 2 * m, dtype=torch.float32, device="cuda")
api.attention_fwd(qs, ks, vs, seg, 0.0, api.ATTN_MID, o_acc=o_acc, lse_acc=lse_acc)
torch.cuda.synchronize()
os.environ["CDSP_TRACE"] = os.path.join(out_dir, "trace_ring.bin")
api.attention_fwd(qs, ks, vs, seg, 0.0, api.ATTN_MID, o_acc=o_acc, lse_acc=lse_acc)
torch.cuda.synchronize()
print("== s=8 ring step (r=3, src=1), MID")
analyze_ctas(os.path.join(out_dir, "trace_ring.bin"), (2 * m // 128) * H)
