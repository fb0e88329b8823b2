"""Copy a refresh_profiles.sh run (gpurun_out/<tag>_*) into profiles/ and print the numbers the
summary quotes.

    python tools/collect_profiles.py r01f [r01]
"""
import json
import os
import shutil
import subprocess
import sys

tag = sys.argv[1]
rnd = sys.argv[2] if len(sys.argv) > 2 else "r01"
src, dst = "gpurun_out", "profiles"
for a, b in ((f"{tag}_bench_c4.json", f"{rnd}_bench_c4.json"),
             (f"{tag}_ref_c4.json", f"{rnd}_bench_reference_c4.json"),
             (f"{tag}_bench_c5.json", f"{rnd}_bench_c5.json"),
             (f"{tag}_launches_c4.csv", f"{rnd}_launches_c4_sweep.csv")):
    shutil.copy(os.path.join(src, a), os.path.join(dst, b))
md, js = [], {}
for rep in (f"{tag}_gram", f"{tag}_solve"):
    path = os.path.join(src, rep + ".ncu-rep")
    md.append(subprocess.run([sys.executable, "tools/ncu_summary.py", path], capture_output=True, text=True).stdout)
    js.update(json.loads(subprocess.run([sys.executable, "tools/ncu_top_json.py", path], capture_output=True,
                                        text=True).stdout))
open(os.path.join(dst, f"{rnd}_ncu_top_kernels.md"), "w").write("".join(md))
json.dump(js, open(os.path.join(dst, f"{rnd}_ncu_top_kernels.json"), "w"), indent=1)
d = json.load(open(os.path.join(dst, f"{rnd}_bench_c4.json")))
print("c4", round(d["value"]), round(d["ms_per_step"], 1), "e2e", round(d["e2e"]["value"]),
      round(d["e2e"]["ms_per_step"], 1), d["clocks"])
print("stages", {k: round(v["ms"], 2) for k, v in d["stages"].items()})
print("kernels", {k: (round(v["ms"], 2), round(v["achieved"], 1), round(v["frac"], 3),
                      round(v.get("fp64_equivalent_tflops", 0), 1)) for k, v in d["kernels"].items()})
print("cpu_baseline", round(d["cpu_baseline"]["value"], 3))
r = json.load(open(os.path.join(dst, f"{rnd}_bench_reference_c4.json")))
print("reference", round(r["value"], 3))
d5 = json.load(open(os.path.join(dst, f"{rnd}_bench_c5.json")))
print("c5", round(d5["value"]), "e2e", round(d5["e2e"]["value"]))
print("ncu", {k: (round(v["duration_ms"], 2), round((v["dram_read_bytes"] + v["dram_write_bytes"]) / 1e9, 2))
              for k, v in js.items()})
print(subprocess.run([sys.executable, "tools/launch_summary.py", os.path.join(dst, f"{rnd}_launches_c4_sweep.csv")],
                     capture_output=True, text=True).stdout)
