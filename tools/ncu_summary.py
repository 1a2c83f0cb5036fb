"""Summarise ncu captures into profiles/*.md (run in the build container).

    python tools/ncu_summary.py gpurun_out/prof_bwd.ncu-rep [more.ncu-rep ...] > profiles/x.md
    python tools/ncu_summary.py --launches gpurun_out/launches.csv
"""

from __future__ import annotations

import csv
import io
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__cycles_active.avg", "SM active cycles (avg)"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor pipe active % (ncu peak)"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_elapsed", "XU/MUFU pipe %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_elapsed", "FMA pipe %"),
    ("l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "smem wavefronts from tensor core %"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "smem wavefronts from LSU %"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 throughput %"),
    ("lts__t_bytes.sum", "L2 bytes (all ops)"),
    ("lts__t_sectors_op_red.sum", "L2 sectors, reductions (red / TMA reduce-add)"),
    ("lts__t_sectors_op_atom.sum", "L2 sectors, atomics"),
    ("lts__t_sectors_op_read.sum", "L2 sectors, reads"),
    ("lts__t_sectors_op_write.sum", "L2 sectors, writes"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput %"),
    ("smsp__inst_executed.sum", "instructions (warp-level)"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__shared_mem_per_block_dynamic", "dynamic smem/block"),
]


def _ncu(args):
    return subprocess.run(["ncu"] + args, capture_output=True, text=True).stdout


def summarize(rep: str) -> str:
    raw = list(csv.reader(io.StringIO(_ncu(["-i", rep, "--page", "raw", "--csv"]))))
    out = [f"## {rep}\n"]
    if len(raw) < 3:
        return out[0] + "(no data)\n"
    hdr, units = raw[0], raw[1]
    for row in raw[2:]:
        d = {h: (u, v) for h, u, v in zip(hdr, units, row)}
        out.append(f"### kernel `{d.get('Kernel Name', ('', '?'))[1][:90]}`\n")
        out.append("| metric | value |\n|---|---|")
        for key, name in METRICS:
            if key in d:
                u, v = d[key]
                out.append(f"| {name} (`{key}`) | {v} {u} |")
        stalls = sorted(((h.replace("smsp__pcsamp_warps_issue_stalled_", ""), float(v or 0))
                         for h, (u, v) in d.items()
                         if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued")
                         and v not in ("", None)), key=lambda x: -x[1])
        tot = sum(v for _, v in stalls) or 1.0
        out.append("\nwarp stall samples (share): " +
                   ", ".join(f"{k} {v / tot:.1%}" for k, v in stalls[:6]) + "\n")
    src = list(csv.reader(io.StringIO(_ncu(["-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"]))))
    if len(src) > 3:
        h = src[2]
        try:
            i_s, i_e = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")

            def num(x):
                try:
                    return float(x)
                except ValueError:
                    return 0.0
            lines = [(num(r[i_s]), r[0], r[1], r[i_e]) for r in src[3:] if r and r[0].isdigit()]
            tot = sum(x[0] for x in lines) or 1.0
            out.append("top source lines by stall samples:\n\n| share | line | executed | source |\n|---|---|---|---|")
            for s, ln, code, ex in sorted(lines, key=lambda x: -x[0])[:12]:
                out.append(f"| {s / tot:.1%} | {ln} | {ex} | `{code.strip()[:80]}` |")
        except ValueError:
            pass
    return "\n".join(out) + "\n"


def launches(path: str) -> str:
    rows = [r for r in csv.reader(open(path)) if r and not r[0].startswith("==")]
    hdr = rows[0]
    i_k, i_m, i_v = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    i_u = hdr.index("Metric Unit")
    agg = {}
    for r in rows[1:]:
        if r[i_m] != "gpu__time_duration.sum":
            continue
        v = float(r[i_v].replace(",", ""))
        if r[i_u] in ("usecond", "us"):
            v /= 1e3
        elif r[i_u] in ("nsecond", "ns"):
            v /= 1e6
        name = r[i_k].split("(")[0][:60]
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += v
    tot = sum(v for _, v in agg.values()) or 1.0
    out = ["| kernel | launches | total ms | ms per launch | share |", "|---|---|---|---|---|"]
    for k, (n, ms) in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append(f"| `{k}` | {n} | {ms:.3f} | {ms / n:.4f} | {ms / tot:.1%} |")
    return "\n".join(out) + "\n"


if __name__ == "__main__":
    if sys.argv[1] == "--launches":
        print(launches(sys.argv[2]))
    else:
        for rep in sys.argv[1:]:
            print(summarize(rep))
