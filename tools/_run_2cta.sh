RP_SOLVE_2CTA=1 timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_cv.py -m gpu -x -q > gpurun_out/s2_pytest.log 2>&1; echo pytest=$? >> gpurun_out/s2_pytest.log
tail -3 gpurun_out/s2_pytest.log
for v in 0 1; do
RP_SOLVE_2CTA=$v python bench.py --steps 5 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/s2.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/s2.json'));print('2cta=$v', round(d['value']), round(d['kernels']['eval_solve']['ms'],2), d['clocks']['sm_mhz'])"
done
