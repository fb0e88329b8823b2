python -m pytest tests -m gpu -q -x > gpurun_out/t.log 2>&1; tail -3 gpurun_out/t.log
python bench.py --steps 5 --warmup 3 --e2e-steps 3 > gpurun_out/b_ob.json 2> gpurun_out/b_ob.err
python -c "import json;d=json.load(open('gpurun_out/b_ob.json'));print(round(d['value']), round(d['e2e']['value']), d['clocks'], {k:round(v['ms'],2) for k,v in d['stages'].items()}, {k:round(v['ms'],2) for k,v in d['kernels'].items()})"
