python -m pytest tests -m gpu -q -x > gpurun_out/t.log 2>&1; tail -n 3 gpurun_out/t.log
for v in 0 1; do
  RP_HOLDOUT_OZAKI=$v python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/ho$v.json 2> gpurun_out/ho$v.err
  python -c "import json;d=json.load(open('gpurun_out/ho$v.json'));print($v, round(d['value']), round(d['e2e']['value']), d['clocks']['sm_mhz'], {k:round(v['ms'],2) for k,v in d['stages'].items()}, {k:round(v['ms'],2) for k,v in d['kernels'].items()})"
done
