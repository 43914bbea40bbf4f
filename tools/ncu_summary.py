"""Summarise ncu evidence into profiles/ (run here, on the CPU host, after gpurun).

  python tools/ncu_summary.py launches <launches.csv> <out.md>     # per-launch durations, kernel shares
  python tools/ncu_summary.py full <report.ncu-rep> <out.md> [key]  # one --set full capture; also writes
                                                                    # profiles/ncu_attn_traffic.json[key]
"""
import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def launches(path, out):
    rows = list(csv.reader(open(path)))
    # ncu --csv log: header row contains "Kernel Name" and "Metric Value"
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[hi]
    ik, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    per = defaultdict(list)
    for r in rows[hi + 1:]:
        if len(r) <= iv or not r[iv]:
            continue
        v = float(r[iv].replace(",", ""))
        unit = r[iu]
        ns = v * {"nsecond": 1, "usecond": 1e3, "msecond": 1e6, "second": 1e9}.get(unit, 1)
        name = r[ik].split("(")[0].replace("void ", "").strip()
        per[name].append(ns)
    total = sum(sum(v) for v in per.values())
    ours = {k: v for k, v in per.items() if k.startswith("cdsp::") or "attn" in k or "decode" in k}
    t_ours = sum(sum(v) for v in ours.values())
    lines = ["| kernel | launches | total ms | avg us | share of all | share of the library's |",
             "|---|---:|---:|---:|---:|---:|"]
    for k, v in sorted(per.items(), key=lambda kv: -sum(kv[1])):
        own = f"{sum(v) / t_ours:.1%}" if k in ours and t_ours else "— (torch: input setup)"
        lines.append(f"| `{k}` | {len(v)} | {sum(v) / 1e6:.3f} | {sum(v) / len(v) / 1e3:.1f} | {sum(v) / total:.1%} | {own} |")
    open(out, "w").write(
        f"# ncu launch list (gpu__time_duration.sum, --clock-control none)\n\nSource: `{os.path.basename(path)}`. "
        "Per-launch times under ncu are cold-cache and serialised: compare SHARES, not absolutes. "
        "torch kernels are the seeded input generation before the timed region.\n\n"
        + "\n".join(lines) + "\n")
    print("\n".join(lines))


WANT = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor pipe active % (elapsed)"),
    ("TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
     "tensor pipe active % (triage 'realtime' counter; undercounts short launches)"),
    ("sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32_sparsity_off.sum", "tensor FLOPs executed (bf16 -> fp32 UTC MMA ops)"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU (MUFU) pipe % of peak"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "FMA pipe % of peak"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "ALU pipe % of peak"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy %"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]


def full(rep, out, key=None):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    lines = ["| metric | value | unit |", "|---|---:|---|"]
    vals = {}
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
        for m, label in WANT:
            if m in hdr:
                i = hdr.index(m)
                vals[m] = (r[i], units[i])
                lines.append(f"| {label} (`{m}`) | {r[i]} | {units[i]} |")
        break
    traffic = None
    if "dram__bytes_read.sum" in vals and "dram__bytes_write.sum" in vals:
        def to_bytes(v, u):
            return float(v.replace(",", "")) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
        traffic = to_bytes(*vals["dram__bytes_read.sum"]) + to_bytes(*vals["dram__bytes_write.sum"])
    open(out, "w").write(f"# ncu --set full: `{name.split('(')[0]}`\n\nReport: `{os.path.basename(rep)}` "
                         "(one launch, --clock-control none).\n\n" + "\n".join(lines) +
                         (f"\n\nDRAM traffic per launch: {traffic:.4g} bytes\n" if traffic else "\n"))
    if key and traffic:
        jp = os.path.join(ROOT, "profiles", "ncu_attn_traffic.json")
        j = json.load(open(jp)) if os.path.exists(jp) else {}
        j[key] = traffic
        json.dump(j, open(jp, "w"), indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3])
    else:
        full(sys.argv[2], sys.argv[3], sys.argv[4] if len(sys.argv) > 4 else None)
