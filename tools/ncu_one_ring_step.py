"""Dev: one warm SP=8 ring-step launch of a 32K chunk (rank 3 attending src 1's shard, MID
merge mode) as the ncu target (--launch-skip 1 --launch-count 1)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from cdsp_inputs import qkv  # noqa: E402
from paper_2511_06247_b200 import api  # noqa: E402

H, D, N, s, r, src = 32, 128, 32768, 8, 3, 1
m = N // (2 * s)
q, k, v = qkv(2 * m, H, H, D, torch.bfloat16, seed=0, device="cuda")
seg = api.segments(2 * m, m, r * m, (2 * s - 1 - r) * m, 2 * m, 0, m, src * m, (2 * s - 1 - src) * m)
o_acc = torch.zeros(2 * m, H, D, dtype=torch.float32, device="cuda")
lse_acc = torch.zeros(H, 2 * m, dtype=torch.float32, device="cuda")
for _ in range(2):
    api.attention_fwd(q, k, v, seg, 0.0, api.ATTN_MID, o_acc=o_acc, lse_acc=lse_acc)
torch.cuda.synchronize()
print("ok")
