"""Dev: one warm s=1 32K causal attention launch (profile target for ncu --launch-skip 1)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from cdsp_inputs import qkv  # noqa: E402
from paper_2511_06247_b200 import api  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
H = 32
q, k, v = qkv(N, H, H, 128, torch.bfloat16, seed=0, device="cuda")
out = torch.empty_like(q)
for _ in range(2):
    api.attention_fwd(q, k, v, api.causal_segments(N, N), 0.0, api.ATTN_ONLY, out=out)
torch.cuda.synchronize()
print("ok")
