timeout 120 ./tools/ozaki_test big 2>&1 | tail -6
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/t.log 2>&1; tail -n 2 gpurun_out/t.log
for v in 1 0; do
  RP_OZAKI_CLUSTER=$v timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/cl$v.json 2> gpurun_out/cl$v.err
  python -c "import json;d=json.load(open('gpurun_out/cl$v.json'));print($v, round(d['value']), round(d['e2e']['value']), d['clocks']['sm_mhz'], {k:round(v['ms'],2) for k,v in d['stages'].items()}, {k:round(v['ms'],2) for k,v in d['kernels'].items()})"
done
