timeout 120 ./tools/ozaki_test big 2>&1 | tail -8
python -m pytest tests -m gpu -q -x 2>&1 | tail -4
for v in 0 1; do
  RP_CHOL_DMMA=$v python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/ch$v.json 2> gpurun_out/ch$v.err
  python -c "import json;d=json.load(open('gpurun_out/ch$v.json'));print($v, round(d['value']), round(d['e2e']['value']), d['stages']['gram']['ms'], d['stages']['factorize'])"
done
