python -m pytest tests/test_gpu_kernels.py tests/test_gpu_cv.py tests/test_gpu_dropin.py tests/test_gpu_exact_cli.py -q -x 2>&1 | tail -3
python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/sv0.json 2> gpurun_out/sv0.err
python -c "import json;d=json.load(open('gpurun_out/sv0.json'));print(round(d['value']), round(d['e2e']['value']), d['stages']['solve'])"
RP_SOLVE_DBG=2 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/sv2.json 2> gpurun_out/sv2.err
python -c "import json;d=json.load(open('gpurun_out/sv2.json'));print('dbg2', round(d['value']), d['stages']['solve'])"
