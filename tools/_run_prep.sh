timeout 120 ./tools/ozaki_test big 2>&1 | tail -4
python -m pytest tests -m gpu -q -x > gpurun_out/t.log 2>&1; tail -n 2 gpurun_out/t.log
python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 3 > gpurun_out/prep.json 2> gpurun_out/prep.err
python -c "import json;d=json.load(open('gpurun_out/prep.json'));print(round(d['value']), round(d['e2e']['value']), d['clocks'], {k:round(v['ms'],2) for k,v in d['stages'].items()}, {k:round(v['ms'],2) for k,v in d['kernels'].items()})"
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"oz_rowexp|oz_slice" --launch-count 6 python bench.py --steps 1 --warmup 0 --e2e-steps 1 --no-cpu-baseline 2>/dev/null | grep -E "oz_|duration" | head -12
