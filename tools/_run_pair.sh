timeout 120 ./tools/ozaki_test | tail -2
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pair_pytest.log 2>&1; echo pytest=$? >> gpurun_out/pair_pytest.log
tail -3 gpurun_out/pair_pytest.log
for ob in 512 768 1024; do
RP_CHOL_OB=$ob python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/pair_c4_$ob.json 2> gpurun_out/pair_c4.err
python -c "import json;d=json.load(open('gpurun_out/pair_c4_$ob.json'));print('ob=$ob', round(d['value']), round(d['e2e']['value']), d['clocks']['sm_mhz'], {k:round(v['ms'],2) for k,v in d['stages'].items()}, {k:round(v['ms'],2) for k,v in d['kernels'].items()})"
done
