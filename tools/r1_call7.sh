python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 300 python tools/bench_decode.py 2>&1 | cut -c1-300
timeout 300 python tools/bench_decode.py --identity-table 2>&1 | cut -c1-300
python - <<'PY'
import torch
x = torch.empty(1 << 30, dtype=torch.bfloat16, device="cuda").normal_()
for f in (lambda: x.sum(), lambda: x.view(-1, 1024).amax(1)):
    for _ in range(3): f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): f()
    e1.record(); torch.cuda.synchronize()
    print("read-only GB/s", 2 * (1 << 30) * 10 / (e0.elapsed_time(e1) * 1e-3) / 1e9)
PY
