"""Dev: run the bench workload's attention kernel back-to-back for a few seconds while
sampling nvidia-smi every 50 ms (SM clock, power, throttle reasons)."""
import subprocess, sys, time, threading, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2511_06247_b200 import api
import cdsp_inputs

L, H, D = 32768, 32, 128
q, k, v = cdsp_inputs.qkv(L, H, H, D, dtype=torch.bfloat16, device="cuda")
out = torch.empty_like(q)
seg = api.causal_segments(L, L)
rows = []
def sample():
    p = subprocess.Popen(["nvidia-smi", "-i", "0", "--query-gpu=clocks.sm,power.draw,clocks_event_reasons.active,temperature.gpu",
                          "--format=csv,noheader,nounits", "-lms", "50"], stdout=subprocess.PIPE, text=True)
    t0 = time.time()
    while time.time() - t0 < float(sys.argv[1]) + 1:
        rows.append(p.stdout.readline().strip())
    p.terminate()
th = threading.Thread(target=sample); th.start()
t0 = time.time(); n = 0
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ev0.record()
while time.time() - t0 < float(sys.argv[1]):
    for _ in range(10):
        api.attention_fwd(q, k, v, seg, 1.0 / D ** 0.5, out=out)
    torch.cuda.synchronize(); n += 10
ev1.record(); torch.cuda.synchronize()
th.join()
fl = 4 * D * H * L * (L + 1) / 2
ms = ev0.elapsed_time(ev1) / n
import statistics
vals = [r.split(",") for r in rows if r.count(",") >= 3]
load = [v for v in vals if float(v[1]) > 600]
clk = statistics.median(float(v[0]) for v in load) if load else float("nan")
pw = statistics.median(float(v[1]) for v in load) if load else float("nan")
tag = os.environ.get("NVCC_APPEND_FLAGS", "")
print(f"[{tag}] {n} launches, {ms:.3f} ms each, {fl / ms / 1e9:.1f} TF/s sustained; under load: sm {clk:.0f} MHz, {pw:.0f} W ({len(load)} samples)")
