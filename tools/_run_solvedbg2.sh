for dbg in 4 0; do
RP_SOLVE_DBG=$dbg python bench.py --steps 3 --warmup 2 --e2e-steps 1 --no-cpu-baseline > gpurun_out/sd_$dbg.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/sd_$dbg.json'));print('dbg=$dbg', round(d['value']), round(d['kernels']['eval_solve']['ms'],2), d['clocks']['sm_mhz'])"
done
