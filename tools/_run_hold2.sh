timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/h2_pytest.log 2>&1; echo pytest=$? >> gpurun_out/h2_pytest.log
tail -3 gpurun_out/h2_pytest.log
python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/h2_c4.json 2> gpurun_out/h2_c4.err
python -c "import json;d=json.load(open('gpurun_out/h2_c4.json'));print(round(d['value']), round(d['e2e']['value']), d['clocks'], {k:round(v['ms'],2) for k,v in d['stages'].items()}, {k:round(v['ms'],2) for k,v in d['kernels'].items()})"
