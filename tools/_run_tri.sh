python -m pytest tests/test_gpu_kernels.py tests/test_gpu_cv.py tests/test_gpu_exact_cli.py -q -x 2>&1 | tail -3
for v in 0 1; do
  RP_HOLDOUT_FULL=$v python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/tri$v.json 2> gpurun_out/tri$v.err
  python -c "import json;d=json.load(open('gpurun_out/tri$v.json'));print($v, round(d['value']), round(d['e2e']['value']), d['stages']['holdout'])"
done
