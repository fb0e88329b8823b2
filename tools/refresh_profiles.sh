#!/bin/bash
# Round-end evidence on one B200 (run through gpurun from the repo root; outputs in gpurun_out/, the ones
# to keep are copied into profiles/ by tools/collect_profiles.py or by hand). Tag: first argument.
# Every step has its own timeout; a number printed under ncu is never a bench value.
tag=${1:-r02}
o=gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > $o/${tag}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $o/${tag}_pytest_gpu.log
timeout 900 python bench.py --steps 5 --warmup 3 > $o/${tag}_bench_c4.json 2> $o/${tag}_bench_c4.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $o/${tag}_bench_reference_c4.json 2> $o/${tag}_ref_c4.err
timeout 900 python bench.py --config c5 --steps 3 --warmup 3 --no-cpu-baseline --no-dropin > $o/${tag}_bench_c5.json 2> $o/${tag}_bench_c5.err
# launch list of exactly one sweep, then full captures of the dominant kernels (never timed)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $o/${tag}_launches_c4.csv \
    python tools/one_sweep.py c4 > $o/${tag}_launch_run.log 2>&1
# full ncu reports stay on the box (/tmp: they exceed what gpurun brings back); their summaries and
# the per-launch DRAM traffic bench.py quotes come back as text, plus the c4 solve report
for cfg in c4 c5; do
  timeout 1200 ncu --set full --import-source on --clock-control none -k regex:oz_syrk -c 1 -o /tmp/${tag}_${cfg}_gram -f \
      python tools/one_sweep.py $cfg > $o/${tag}_${cfg}_ncu_gram.log 2>&1
  timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"eval_solve|oz_dotb" -c 5 \
      -o /tmp/${tag}_${cfg}_solve -f python tools/one_sweep.py $cfg > $o/${tag}_${cfg}_ncu_solve.log 2>&1
  python tools/ncu_summary.py /tmp/${tag}_${cfg}_gram.ncu-rep > $o/${tag}_ncu_${cfg}_gram.md 2>&1
  python tools/ncu_summary.py /tmp/${tag}_${cfg}_solve.ncu-rep > $o/${tag}_ncu_${cfg}_solve.md 2>&1
done
python tools/ncu_top_json.py c4=/tmp/${tag}_c4_gram.ncu-rep c4=/tmp/${tag}_c4_solve.ncu-rep \
    c5=/tmp/${tag}_c5_gram.ncu-rep c5=/tmp/${tag}_c5_solve.ncu-rep > $o/${tag}_ncu_top_kernels.json 2>&1
cp /tmp/${tag}_c4_solve.ncu-rep $o/ 2>/dev/null
tail -2 $o/${tag}_pytest_gpu.log
python - "$tag" <<'EOF'
import json, sys
tag = sys.argv[1]
for name in (f"gpurun_out/{tag}_bench_c4.json", f"gpurun_out/{tag}_bench_c5.json", f"gpurun_out/{tag}_bench_reference_c4.json"):
    try:
        d = json.loads(open(name).read().strip().splitlines()[-1])
    except Exception as e:  # noqa: BLE001
        print(name, "unreadable", e)
        continue
    print(name, round(d["value"], 1), round(d["e2e"]["value"], 1), d.get("clocks"),
          {k: round(v["ms"], 2) for k, v in d.get("stages", {}).items()}, d.get("roofline", {}).get("frac"))
EOF
