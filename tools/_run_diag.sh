timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/t.log 2>&1; tail -n 2 gpurun_out/t.log
python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 3 > gpurun_out/dg.json 2> gpurun_out/dg.err
python -c "import json;d=json.load(open('gpurun_out/dg.json'));print(round(d['value']), round(d['e2e']['value']), d['clocks']['sm_mhz'], {k:round(v['ms'],2) for k,v in d['stages'].items()})"
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:potrf_diag --launch-count 3 python bench.py --steps 1 --warmup 0 --e2e-steps 1 --no-cpu-baseline 2>/dev/null | grep -E "duration" | head -3
