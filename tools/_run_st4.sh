timeout 120 ./tools/ozaki_test big 2>&1 | tail -3
for v in 0 1; do
  RP_OZAKI_CLUSTER=$v timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/st4_$v.json 2> gpurun_out/st4_$v.err
  python -c "import json;d=json.load(open('gpurun_out/st4_$v.json'));print($v, round(d['value']), round(d['e2e']['value']), d['clocks']['sm_mhz'], {k:round(v['ms'],2) for k,v in d['stages'].items()}, {k:round(v['ms'],2) for k,v in d['kernels'].items()})"
done
