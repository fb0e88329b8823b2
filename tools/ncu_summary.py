"""Summarise an ncu report (--set full, -lineinfo build) into markdown for profiles/.

    python tools/ncu_summary.py gpurun_out/top_r01.ncu-rep > profiles/r01_ncu_top.md

Per kernel: duration, DMMA / FP64 pipe utilisation, issue activity, DRAM traffic, the warp
stall breakdown and the source lines with the most stall samples.
"""

import csv
import io
import subprocess
import sys
from collections import defaultdict

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active", "DMMA pipe %"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "DFMA pipe %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
     "tensor pipe (tcgen05) active %"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 throughput %"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate %"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput %"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("launch__registers_per_thread", "registers"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]


def ncu(*args):
    return subprocess.run(["ncu", *args], capture_output=True, text=True).stdout


def main(rep):
    raw = list(csv.reader(io.StringIO(ncu("-i", rep, "--page", "raw", "--csv"))))
    h, u = raw[0], raw[1]
    print(f"# ncu summary: `{rep.split('/')[-1]}`\n")
    for idx, r in enumerate(raw[2:]):
        name = r[h.index("Kernel Name")]
        print(f"## {idx}: `{name[:100]}`\n")
        print("| metric | value |\n|---|---|")
        for k, label in KEYS:
            if k in h:
                print(f"| {label} | {r[h.index(k)]} {u[h.index(k)]} |")
        st = [(k.replace("smsp__pcsamp_warps_issue_stalled_", ""), float(v)) for k, v in zip(h, r)
              if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")
              and v not in ("", "nan", "-nan")]
        tot = sum(v for _, v in st) or 1.0
        top = sorted(st, key=lambda x: -x[1])[:8]
        print("\nstalls: " + ", ".join(f"{k} {v / tot * 100:.1f}%" for k, v in top) + "\n")
        src = list(csv.reader(io.StringIO(ncu("-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                                               "--launch-skip", str(idx), "--launch-count", "1"))))
        agg, text = defaultdict(float), {}
        cur, col = None, None
        for row in src:
            if row and row[0] == "File Path":
                cur = row[1].split("/")[-1]
            elif row and row[0] == "Line No":
                col = row.index("Warp Stall Sampling (All Samples)")
            elif row and row[0].isdigit() and cur and col is not None and len(row) > col:
                try:
                    agg[(cur, int(row[0]))] += float(row[col] or 0)
                except ValueError:
                    continue
                text[(cur, int(row[0]))] = row[1].strip()
        t = sum(agg.values()) or 1.0
        print("| stall share | source line |\n|---|---|")
        for key, v in sorted(agg.items(), key=lambda x: -x[1])[:10]:
            print(f"| {v / t * 100:.1f}% | `{key[0]}:{key[1]}` {text[key][:80]} |")
        print()


if __name__ == "__main__":
    main(sys.argv[1])
