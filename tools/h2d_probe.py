"""Dev: host->device bandwidth from pinned memory for the e2e leg's 805 MB of q/k/v: one stream
vs one stream per tensor vs 8 pieces over 4 streams, with and without a concurrent 268 MB D2H."""
import time

import torch

dev = torch.device("cuda:0")
n = 32768 * 32 * 128
hs = [torch.empty(n, dtype=torch.bfloat16).pin_memory() for _ in range(3)]
ds = [torch.empty(n, dtype=torch.bfloat16, device=dev) for _ in range(3)]
ho = torch.empty(n, dtype=torch.bfloat16).pin_memory()
do = torch.empty(n, dtype=torch.bfloat16, device=dev)
streams = [torch.cuda.Stream() for _ in range(5)]


def run(nstreams, pieces, with_d2h):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    cur = torch.cuda.current_stream()
    e0.record(cur)
    for s in streams:
        s.wait_stream(cur)
    jobs = []
    for h, d in zip(hs, ds):
        step = n // pieces
        for i in range(pieces):
            jobs.append((h[i * step:(i + 1) * step], d[i * step:(i + 1) * step]))
    for i, (h, d) in enumerate(jobs):
        with torch.cuda.stream(streams[i % nstreams]):
            d.copy_(h, non_blocking=True)
    if with_d2h:
        with torch.cuda.stream(streams[4]):
            ho.copy_(do, non_blocking=True)
    for s in streams:
        cur.wait_stream(s)
    e1.record(cur)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    return 3 * n * 2 / (ms * 1e-3) / 1e9, ms


for cfg in [(1, 1, False), (3, 1, False), (4, 8, False), (1, 1, True), (3, 1, True), (4, 8, True)]:
    r = [run(*cfg) for _ in range(5)]
    best = max(r)
    print(f"streams={cfg[0]} pieces/tensor={cfg[1]} d2h={cfg[2]}: H2D {best[0]:.1f} GB/s ({best[1]:.2f} ms)")
