for dbg in 0 1 2 4; do
RP_SOLVE_DBG=$dbg python bench.py --steps 3 --warmup 2 --e2e-steps 1 --no-cpu-baseline > gpurun_out/sd.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/sd.json'));print('dbg=$dbg', round(d['kernels']['eval_solve']['ms'],2), d['clocks']['sm_mhz'])"
done
