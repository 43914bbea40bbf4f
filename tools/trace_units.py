"""Dev: timelines of the persistent attn_tc kernel (build with CDSP_KTRACE=1).
(a) s=1 32K causal (ONLY), (b) one SP=8 ring step (r=3, src=1, MID) of the 32K chunk.
Per unit (globaltimer ns): published, first S read, loop end, epilogue end; per tile of
CTAs 0-3 (clock64): PV / S issue, S seen, m ready, exps done, P arrive.
usage: python tools/trace_units.py <out_dir>"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def analyze(path, n_units):
    raw = np.fromfile(path, dtype=np.uint64)
    c = raw[:65536 * 8].reshape(-1, 8)[:n_units].astype(np.int64)
    pub, end, sm, nu, first_s, loop_end, epi = c[:, 0], c[:, 1], c[:, 2], c[:, 3], c[:, 5], c[:, 6], c[:, 7]
    ok = nu > 0
    t0 = pub[ok].min()
    span = end[ok].max() - t0
    print(f"kernel span {span / 1e3:.1f} us, {ok.sum()} non-empty units, SMs {len(set(sm[ok].tolist()))}")
    for name, a_, b_ in (("pub->first S", pub, first_s), ("first S->loop end", first_s, loop_end),
                         ("loop end->epi end", loop_end, epi)):
        x = (b_ - a_)[ok] / 1e3
        print(f"  {name:20s} median {np.median(x):8.2f} us  p90 {np.percentile(x, 90):8.2f}")
    # per SM: boundary = previous unit's loop end -> this unit's first S read
    gaps, tails = [], []
    for s_ in set(sm[ok].tolist()):
        idx = np.nonzero(ok & (sm == s_))[0]
        o = idx[np.argsort(first_s[idx])]
        gaps += list(first_s[o[1:]] - loop_end[o[:-1]])
        tails.append(end[ok].max() - epi[o[-1]])
    print(f"  boundary (loop end -> next first S) median {np.median(gaps):.0f} ns mean {np.mean(gaps):.0f} ns")
    print(f"  SM tail idle median {np.median(tails) / 1e3:.1f} us, max {np.max(tails) / 1e3:.1f} us")
    b, a = np.polyfit(nu[ok], (loop_end - first_s)[ok], 1)
    print(f"  fit loop time: {a / 1e3:.2f} us + {b:.1f} ns per tile")
    # where the span goes, averaged over SMs: tiles (loop), unit boundaries, epilogues, tail
    n_sm = len(set(sm[ok].tolist()))
    loop_t = (loop_end - first_s)[ok].sum() / n_sm / 1e3
    tiles_per_sm = nu[ok].sum() / n_sm
    print(f"  per SM: {tiles_per_sm:.0f} tiles, loop {loop_t:.1f} us ({loop_t * 1e3 / max(tiles_per_sm, 1):.0f} ns/tile),"
          f" units {ok.sum() / n_sm:.1f}, boundary total {np.sum(gaps) / n_sm / 1e3:.1f} us,"
          f" tail {np.mean(tails) / 1e3:.1f} us, span {span / 1e3:.1f} us")
    it = raw[65536 * 8:].reshape(4, 512, 16).astype(np.int64)
    d = it[0]
    n = int((d[:, 8] > 0).sum())
    pv = d[:n, 8]
    dpv = np.diff(pv)
    med = np.median(dpv)
    print(f"  CTA0 PV issue period median {med:.0f} clk (ideal 1024); intervals > 2x median: "
          f"{(dpv > 2 * med).sum()} totalling {dpv[dpv > 2 * med].sum():.0f} clk of {pv[-1] - pv[0]:.0f}")
    g = np.arange(n) & 1
    s_seen = d[np.arange(n), 4 * g]
    m_ready = d[np.arange(n), 4 * g + 1]
    exps = d[np.arange(n), 4 * g + 2]
    p_arr = d[np.arange(n), 4 * g + 3]
    for name, x in (("S seen->m ready", m_ready - s_seen), ("m ready->exps done", exps - m_ready),
                    ("exps->P arrive", p_arr - exps), ("P arrive->PV issue", pv - p_arr),
                    ("S issue->S seen", s_seen[3:] - d[3:n, 9]), ("MMA V wait", d[:n, 11] - d[:n, 10]),
                    ("MMA P wait (after V)", pv - d[:n, 11]), ("K load->S issue", d[3:n, 9] - d[3:n, 15]),
                    ("V load->PV issue", pv[3:] - d[3:n, 14])):
        print(f"  {name:20s} median {np.median(x):7.0f}  p90 {np.percentile(x, 90):7.0f}")
    big = np.nonzero(dpv > 2 * med)[0][:6]
    for k in big:
        print(f"   stall before tile {k + 1}: {dpv[k]} clk; P({k + 1}) arrive - PV({k}) = {p_arr[k + 1] - pv[k]}, "
              f"S({k + 1}) seen - PV({k}) = {s_seen[k + 1] - pv[k]}, S({k+1}) issue - PV({k}) = {d[k + 1, 9] - pv[k]}")


if __name__ == "__main__":
    import torch
    from cdsp_inputs import qkv
    from paper_2511_06247_b200 import api
    out_dir = sys.argv[1]
    H, D, N = 32, 128, 32768
    q, k, v = qkv(N, H, H, D, torch.bfloat16, seed=0, device="cuda")
    out = torch.empty_like(q)
    api.attention_fwd(q, k, v, api.causal_segments(N, N), 0.0, api.ATTN_ONLY, out=out)
    torch.cuda.synchronize()
    os.environ["CDSP_TRACE"] = os.path.join(out_dir, "trace_s1.bin")
    api.attention_fwd(q, k, v, api.causal_segments(N, N), 0.0, api.ATTN_ONLY, out=out)
    torch.cuda.synchronize()
    del os.environ["CDSP_TRACE"]
    print("== s=1 32K causal")
    analyze(os.path.join(out_dir, "trace_s1.bin"), 8192)
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
    analyze(os.path.join(out_dir, "trace_ring.bin"), (2 * m // 128) * H)
    # fused ring launches of ranks 0 and 7 (all 8 blocks in one launch)
    sh = [(api.zigzag_gather(q, s, x), api.zigzag_gather(k, s, x), api.zigzag_gather(v, s, x)) for x in range(s)]
    acc = torch.empty(2 * m, H, D, dtype=torch.float32, device="cuda")
    lacc = torch.empty(H, 2 * m, dtype=torch.float32, device="cuda")
    ranks_env = os.environ.get("TRACE_RANKS")
    combos = [(int(x), True) for x in ranks_env.split(",")] if ranks_env else [(0, False), (0, True), (7, False), (7, True)]
    for r, split in combos:
        srcs = [(r - st) % s for st in range(s)]
        segs = [api.segments(2 * m, m, r * m, (2 * s - 1 - r) * m, 2 * m, 0, m, x * m, (2 * s - 1 - x) * m) for x in srcs]
        outr = torch.empty_like(sh[r][0])
        args = (sh[r][0], [sh[x][1] for x in srcs], [sh[x][2] for x in srcs], segs, 0.0, api.ATTN_ONLY)
        kw = dict(out=outr, o_acc=acc, lse_acc=lacc) if split else dict(out=outr)
        api.attention_fwd_blocks(*args, **kw)
        torch.cuda.synchronize()
        os.environ["CDSP_TRACE"] = os.path.join(out_dir, f"trace_fused_r{r}.bin")
        api.attention_fwd_blocks(*args, **kw)
        torch.cuda.synchronize()
        del os.environ["CDSP_TRACE"]
        print(f"== s=8 fused ring launch, rank {r}{' (split units)' if split else ''}")
        analyze(os.path.join(out_dir, f"trace_fused_r{r}.bin"), 65536)
