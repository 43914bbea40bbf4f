"""Dev: burst vs sustained rate of the s=1 kernel (32K MHA chunk, one launch per step): 60
launches back to back, each CUDA-event timed; prints TF/s of launches 1-5 and 40-59, and the
SM clock / power sampled by NVML during the run."""
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from cdsp_inputs import qkv  # noqa: E402
from paper_2511_06247_b200 import api  # noqa: E402

L, H, D = 32768, 32, 128
dev = torch.device("cuda:0")
flops = 4.0 * D * H * L * (L + 1) / 2
q, k, v = qkv(L, H, H, D, torch.bfloat16, seed=0, device=dev)
seg = api.causal_segments(L, L)
out = torch.empty_like(q)
samples = []
stop = False


def sampler():
    import pynvml
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(0)
    while not stop:
        samples.append((pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM), pynvml.nvmlDeviceGetPowerUsage(h) / 1000,
                        pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)))
        time.sleep(0.005)


n = 60
api.attention_fwd(q, k, v, seg, 0.0, api.ATTN_ONLY, out=out)
torch.cuda.synchronize()
time.sleep(1.0)  # cool down
th = threading.Thread(target=sampler)
th.start()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(n + 1)]
ev[0].record()
for i in range(n):
    api.attention_fwd(q, k, v, seg, 0.0, api.ATTN_ONLY, out=out)
    ev[i + 1].record()
torch.cuda.synchronize()
stop = True
th.join()
tf = [flops / (ev[i].elapsed_time(ev[i + 1]) * 1e-3) / 1e12 for i in range(n)]
b = sum(tf[1:6]) / 5
s = sum(tf[40:60]) / 20
clk = [c for c, p, r in samples]
pw = [p for c, p, r in samples]
reasons = {}
for c, p, r in samples:
    reasons[hex(r)] = reasons.get(hex(r), 0) + 1
print("NVML reasons bitmask counts:", reasons, " clocks:", clk[:80])
print(f"burst(1-5) {b:.0f} sustained(40-59) {s:.0f} TF/s; sm clock min/median {min(clk)}/{sorted(clk)[len(clk)//2]} MHz; "
      f"power max {max(pw):.0f} W; first {' '.join(f'{x:.0f}' for x in tf[:12])}")
