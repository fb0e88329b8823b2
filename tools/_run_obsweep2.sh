for ob in 512 768 1024 1536; do for g in 4; do
RP_CHOL_OB=$ob RP_CHOL_GROUPS=$g python bench.py --steps 3 --warmup 2 --e2e-steps 1 --no-cpu-baseline > gpurun_out/ob2_${ob}_$g.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/ob2_${ob}_$g.json'));print('ob=$ob g=$g', round(d['value']), round(d['stages']['factorize']['ms'],2), round(d['stages']['gram']['ms'],2), round(d['ms_per_step'],2))"
done; done
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/oz_pytest.log 2>&1; echo pytest=$? >> gpurun_out/oz_pytest.log
tail -3 gpurun_out/oz_pytest.log
