timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/ea_pytest.log 2>&1; echo pytest=$? >> gpurun_out/ea_pytest.log
tail -3 gpurun_out/ea_pytest.log
python tools/e2e_probe.py > gpurun_out/ea_probe.log 2>&1; cat gpurun_out/ea_probe.log
python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ea_c4.json 2> gpurun_out/ea_c4.err
python -c "import json;d=json.load(open('gpurun_out/ea_c4.json'));print(round(d['value']), round(d['e2e']['value']), d['e2e']['ms_per_step'], {k:round(v['ms'],2) for k,v in d['stages'].items()})"
