python -m pytest tests -m gpu -q -x 2>&1 | tail -4
for v in 0 1; do
  RP_GRAM_DMMA=$v python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/oz$v.json 2> gpurun_out/oz$v.err
  python -c "import json;d=json.load(open('gpurun_out/oz$v.json'));print($v, round(d['value']), round(d['e2e']['value']), d['stages']['gram'])"
done
