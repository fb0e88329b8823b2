#!/bin/bash
# Round-end evidence on one B200 (run through gpurun from the repo root; outputs in gpurun_out/,
# the ones to keep are copied into profiles/ by hand). Tag: first argument (default r01).
tag=${1:-r01}
python bench.py --steps 5 --warmup 3 > gpurun_out/${tag}_bench_c4.json 2> gpurun_out/${tag}_bench_c4.err
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${tag}_ref_c4.json 2> gpurun_out/${tag}_ref_c4.err
python bench.py --config c5 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/${tag}_bench_c5.json 2> gpurun_out/${tag}_bench_c5.err
# launch list of exactly one sweep, then full captures of the dominant kernels (never timed)
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${tag}_launches_c4.csv \
    python tools/one_sweep.py > gpurun_out/${tag}_launch_run.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:oz_syrk -c 1 -o gpurun_out/${tag}_gram \
    python tools/one_sweep.py > gpurun_out/${tag}_ncu_gram.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"eval_solve|oz_dotb" -c 3 -o gpurun_out/${tag}_solve \
    python tools/one_sweep.py > gpurun_out/${tag}_ncu_solve.log 2>&1
python -c "import json;d=json.load(open('gpurun_out/${tag}_bench_c4.json'));print(round(d['value']), round(d['e2e']['value']), d['clocks'], {k:round(v['ms'],2) for k,v in d['stages'].items()})"
head -c 300 gpurun_out/${tag}_ref_c4.json; echo
python -c "import json;d=json.load(open('gpurun_out/${tag}_bench_c5.json'));print(round(d['value']), round(d['e2e']['value']))"
