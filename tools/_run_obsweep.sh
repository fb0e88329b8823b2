for ob in 512 768 1024 1536; do for g in 4 8; do
RP_CHOL_OB=$ob RP_CHOL_GROUPS=$g python bench.py --steps 3 --warmup 2 --e2e-steps 1 --no-cpu-baseline > gpurun_out/ob_$ob_$g.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/ob_$ob_$g.json'));print('ob=$ob g=$g', round(d['value']), round(d['stages']['factorize']['ms'],2), round(d['ms_per_step'],2))"
done; done
