for ob in 384 512 640 768 1024; do for g in 4 6 8; do
RP_CHOL_OB=$ob RP_CHOL_GROUPS=$g python bench.py --steps 5 --warmup 2 --e2e-steps 1 --no-cpu-baseline > gpurun_out/ob4.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/ob4.json'));print('ob=$ob g=$g', round(d['value']), round(d['stages']['factorize']['ms'],2), round(d['ms_per_step'],2), d['clocks']['sm_mhz'])"
done; done
