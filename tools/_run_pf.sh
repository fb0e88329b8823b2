RP_CHOL_GROUPS=1 python tools/timeline.py c4 gpurun_out/tl_pf.txt > /dev/null 2>&1; python tools/chol_calls.py gpurun_out/tl_pf.txt
python bench.py --steps 5 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/pf.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/pf.json'));print(round(d['value']), d['clocks']['sm_mhz'], {k:round(v['ms'],2) for k,v in d['stages'].items()})"
