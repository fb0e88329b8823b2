for cfg in "4 1536" "2 1536" "8 1536" "4 1024" "4 2048" "6 1536"; do
  set -- $cfg
  RP_CHOL_GROUPS=$1 RP_CHOL_OB=$2 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/sw.json 2> gpurun_out/sw.err
  python -c "import json;d=json.load(open('gpurun_out/sw.json'));print('$1 $2', round(d['value']), d['clocks']['sm_mhz'], round(d['stages']['factorize']['ms'],2))"
done
