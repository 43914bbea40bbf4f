"""Dev tool: run one block-attention launch with the in-kernel timeline enabled
(CDSP_TRACE=<file>) and print per-iteration event deltas of the first CTAs."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
SLOTS = ["S0", "Sfree0", "exp0", "P0", "S1", "Sfree1", "exp1", "P1", "m:QK0", "m:QK1", "m:PV0", "m:PV1"]


def run(path, N=32768, H=32, Hkv=32):
    import torch
    from cdsp_inputs import qkv
    from paper_2511_06247_b200 import api
    q, k, v = (t.cuda() for t in qkv(N, H, Hkv, 128, torch.bfloat16, seed=0, device="cuda"))
    out = torch.empty_like(q)
    api.attention_fwd(q, k, v, api.causal_segments(N, N), 0.0, api.ATTN_ONLY, out=out)  # warm (no trace)
    os.environ["CDSP_TRACE"] = path
    torch.cuda.synchronize()


def analyze_ctas(path, n_cta):
    raw = np.fromfile(path, dtype=np.uint64)
    c = raw[:65536 * 8].reshape(-1, 8)[:n_cta].astype(np.int64)
    start, end, sm, nu = c[:, 0], c[:, 1], c[:, 2], c[:, 3]
    setup, firstS, loopend, epiend = c[:, 4], c[:, 5], c[:, 6], c[:, 7]
    for name, a_, b_ in (("start->setup", start, setup), ("setup->first S", setup, firstS),
                         ("first S->loop end", firstS, loopend), ("loop end->epi end", loopend, epiend),
                         ("epi end->CTA end", epiend, end)):
        x = (b_ - a_) / 1e3
        print(f"{name:20s} median {np.median(x):8.2f} us  p90 {np.percentile(x, 90):8.2f}  max {x.max():8.2f}")
    t0 = start.min()
    span = end.max() - t0
    dur = end - start
    print(f"kernel span {span/1e3:.1f} us over {n_cta} CTAs; SMs used {len(set(sm.tolist()))}")
    busy = np.zeros(int(sm.max()) + 1)
    for i in range(n_cta):
        busy[sm[i]] += dur[i]
    print(f"SM busy fraction: mean {busy.mean()/span:.3f} min {busy.min()/span:.3f}")
    per_it = dur / np.maximum(nu, 1)
    print(f"ns per used KV tile: median {np.median(per_it):.1f}; by size quartile:",
          [round(float(np.median(per_it[(nu >= a) & (nu < b)])), 1) for a, b in ((0, 64), (64, 256), (256, 1024), (1024, 10**9)) if ((nu >= a) & (nu < b)).any()])
    # fixed per-CTA overhead from a linear fit dur = a + b * nu
    b, a = np.polyfit(nu, dur, 1)
    print(f"fit: per-CTA overhead {a/1e3:.2f} us, per KV tile {b:.1f} ns")
    # gaps between consecutive CTAs on the same SM
    gaps = []
    for s_ in set(sm.tolist()):
        idx = np.nonzero(sm == s_)[0]
        o = idx[np.argsort(start[idx])]
        gaps += list(start[o[1:]] - end[o[:-1]])
    print(f"gap between CTAs on an SM: median {np.median(gaps):.0f} ns, mean {np.mean(gaps):.0f} ns")
    last = end.max()
    print(f"tail: SMs idle at end (time from SM's last CTA end to kernel end) median {np.median([last - end[sm == s_].max() for s_ in set(sm.tolist())])/1e3:.1f} us")


def analyze_iters(path):
    raw = np.fromfile(path, dtype=np.uint64)
    t = raw[65536 * 8:].reshape(4, 512, 16).astype(np.int64)
    names = {0: "t0 S", 1: "t0 bar", 2: "t0 P", 4: "t1 S", 5: "t1 P", 8: "t0 prePV", 9: "t0 postQK"}
    d = t[0]
    base = d[0, 0]
    print("it  " + " ".join(f"{names[k]:>8}" for k in names))
    for it in range(0, 14):
        print(f"{it:3d} " + " ".join(f"{(d[it, k] - base) if d[it, k] else -1:8d}" for k in names))
    x = d[8:200]
    print("period (t0 S->S)", np.median(np.diff(x[:, 0])), " t1:", np.median(np.diff(x[:, 4])))
    for nm, a_, b_ in (("t0 S->bar", 0, 1), ("t0 bar->P", 1, 2), ("t1 S->P", 4, 5), ("t0 P->prePV", 2, 8),
                       ("t0 prePV->postQK", 8, 9)):
        v = x[:, b_] - x[:, a_]
        print(f"{nm:16s} median {np.median(v):7.0f} p90 {np.percentile(v, 90):7.0f}")
    v = d[9:201, 0] - x[:, 9]
    print(f"t0 postQK->S(next) median {np.median(v):7.0f}")


def analyze(path):
    t = np.fromfile(path, dtype=np.uint64)[:4 * 256 * 16].reshape(4, 256, 16).astype(np.int64)
    cta = 0
    base = t[cta, 0, 0]
    print("it   " + " ".join(f"{x:>7}" for x in SLOTS))
    for it in range(0, 24):
        row = t[cta, it, :12]
        print(f"{it:3d} " + " ".join(f"{(x - base) if x else -1:7d}" for x in row))
    print("MMA warp: pre/post issue stamps (relative to pre-QK0 of the iteration)")
    for it in range(10, 16):
        r = t[cta, it]
        b0 = r[12]
        print(it, "preQK0 0", "postQK0", r[8] - b0, "preQK1", r[13] - b0, "postQK1", r[9] - b0, "prePV0", r[14] - b0,
              "postPV0", r[10] - b0, "prePV1", r[15] - b0, "postPV1", r[11] - b0, "next preQK0", t[cta, it + 1, 12] - b0)
    d = t[cta, 10:200]
    per = np.diff(d[:, 10])
    print("PV0 issue period median", np.median(per), " (ideal 1024 = 4 x 256-clk GEMMs)")
    for name, a_, b_ in (("S0 seen->Sfree0", 0, 1), ("Sfree0->exp0 done", 1, 2), ("exp0->P0 arrive", 2, 3),
                         ("S1 seen->Sfree1", 4, 5), ("Sfree1->exp1", 5, 6), ("exp1->P1", 6, 7),
                         ("P0 arrive->PV0 issued", 3, 10), ("P1 arrive->PV1 issued", 7, 11),
                         ("QK0 issued->S0 seen(next)", 8, None)):
        if b_ is None:
            x = t[cta, 11:201, 0] - d[:, 8]
        else:
            x = d[:, b_] - d[:, a_]
        print(f"{name:28s} median {np.median(x):8.0f}  p10 {np.percentile(x, 10):8.0f}  p90 {np.percentile(x, 90):8.0f}")


if __name__ == "__main__":
    if sys.argv[1] == "run":
        import torch
        from cdsp_inputs import qkv
        from paper_2511_06247_b200 import api
        N, H = 32768, 32
        q, k, v = (t.cuda() for t in qkv(N, H, H, 128, torch.bfloat16, seed=0))
        out = torch.empty_like(q)
        api.attention_fwd(q, k, v, api.causal_segments(N, N), 0.0, api.ATTN_ONLY, out=out)
        torch.cuda.synchronize()
        print("ok")
    else:
        analyze_iters(sys.argv[2])
        analyze_ctas(sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 4096)
