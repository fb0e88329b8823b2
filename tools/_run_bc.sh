python -m pytest tests -m gpu -q -x > gpurun_out/t.log 2>&1; tail -n 2 gpurun_out/t.log
python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 3 > gpurun_out/bc.json 2> gpurun_out/bc.err
python -c "import json;d=json.load(open('gpurun_out/bc.json'));print(round(d['value']), round(d['e2e']['value']), d['clocks']['sm_mhz'], {k:round(v['ms'],2) for k,v in d['stages'].items()})"
