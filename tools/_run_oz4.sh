python -m pytest tests/test_gpu_kernels.py -q -x -k "potrf or gram" 2>&1 | tail -2
for v in 0 1; do
  RP_CHOL_OZAKI=$v python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/c4oz$v.json 2> gpurun_out/c4oz$v.err
  python -c "import json;d=json.load(open('gpurun_out/c4oz$v.json'));print($v, round(d['value']), round(d['e2e']['value']), d['clocks']['sm_mhz'], {k:round(v['ms'],2) for k,v in d['stages'].items()}, round(d['kernels']['oz_syrk']['ms'],2))"
done
