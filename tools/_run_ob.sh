python -m pytest tests -m gpu -q -x 2>&1 | tail -2
for ob in 512 768 1024 1536 2048; do
  RP_CHOL_OB=$ob python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ob$ob.json 2> gpurun_out/ob$ob.err
  python -c "import json;d=json.load(open('gpurun_out/ob$ob.json'));print($ob, round(d['value']), d['clocks']['sm_mhz'], {k:round(v['ms'],2) for k,v in d['stages'].items()})"
done
