timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gp_pytest.log 2>&1; echo pytest=$? >> gpurun_out/gp_pytest.log
tail -3 gpurun_out/gp_pytest.log
python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/gp_c4.json 2> gpurun_out/gp_c4.err
python -c "import json;d=json.load(open('gpurun_out/gp_c4.json'));print(round(d['value']), round(d['e2e']['value']), d['clocks']['sm_mhz'], {k:round(v['ms'],2) for k,v in d['stages'].items()}, {k:round(v['ms'],2) for k,v in d['kernels'].items()})"
python tools/timeline.py c4 gpurun_out/timeline_c4d.txt > gpurun_out/timeline_d.log 2>&1; head -3 gpurun_out/timeline_d.log
