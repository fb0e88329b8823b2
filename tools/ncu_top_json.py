"""Per-launch DRAM traffic and duration of the dominant kernels from an `ncu --set full` report,
as the JSON bench.py reads for roofline.traffic (profiles/rNN_ncu_top_kernels.json).

    python tools/ncu_top_json.py c4=gpurun_out/c4_top.ncu-rep [c5=...] > profiles/r02_ncu_top_kernels.json

Several reports of one config (config=rep, repeated) merge; the output is {config: {kernel: {...}}}.
"""

import csv
import io
import json
import subprocess
import sys

KEYS = {"oz_syrk_kernel": "oz_syrk", "oz_syrk_pair_kernel": "oz_syrk", "eval_solve_kernel": "eval_solve", "32, 3>": "holdout_gemm", "oz_dotb_kernel": "oz_holdout", "oz_dotb_pair_kernel": "oz_holdout"}


def one(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]

    def val(r, k):
        v = float(r[h.index(k)].replace(",", ""))
        u = units[h.index(k)]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-6, "us": 1e-3, "ms": 1.0,
                 "msecond": 1.0, "usecond": 1e-3, "nsecond": 1e-6}.get(u, 1.0)
        return v * scale

    res = {}
    # the fused solve's split plan adds small tail launches beside the main ones: keep the largest grid
    gi = h.index("launch__grid_size") if "launch__grid_size" in h else None
    solve_grid = max((float(r[gi].replace(",", "")) for r in rows[2:] if "eval_solve_kernel" in r[h.index("Kernel Name")]),
                     default=0.0) if gi is not None else 0.0
    for r in rows[2:]:
        name = r[h.index("Kernel Name")]
        if gi is not None and "eval_solve_kernel" in name and float(r[gi].replace(",", "")) < solve_grid:
            continue
        for pat, key in KEYS.items():
            if pat in name:
                e = res.setdefault(key, {"launches": 0, "dram_read_bytes": 0.0, "dram_write_bytes": 0.0,
                                         "duration_ms": 0.0, "kernel": name[:120]})
                e["launches"] += 1
                e["dram_read_bytes"] += val(r, "dram__bytes_read.sum")
                e["dram_write_bytes"] += val(r, "dram__bytes_write.sum")
                e["duration_ms"] += val(r, "gpu__time_duration.sum")
    for e in res.values():  # per launch
        n = e["launches"]
        e["dram_read_bytes"] /= n
        e["dram_write_bytes"] /= n
        e["duration_ms"] /= n
        for k in ("dram_read_bytes", "dram_write_bytes"):  # ncu reports n/a for some long kernels: null, not NaN
            if e[k] != e[k]:
                e[k] = None
    return res


def main(pairs):
    res = {}
    for pair in pairs:
        cfg, rep = pair.split("=", 1)
        res.setdefault(cfg, {}).update(one(rep))
    json.dump(res, sys.stdout, indent=1)
    print()


if __name__ == "__main__":
    main(sys.argv[1:])
