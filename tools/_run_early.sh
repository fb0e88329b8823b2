timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/t.log 2>&1; tail -n 3 gpurun_out/t.log
python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 3 > gpurun_out/early.json 2> gpurun_out/early.err
python -c "import json;d=json.load(open('gpurun_out/early.json'));print(round(d['value']), round(d['e2e']['value']), d['e2e']['ms_per_step'], d['clocks']['sm_mhz'])"
