for v in 0 4; do
  RP_SOLVE_DBG=$v python bench.py --steps 3 --warmup 2 --no-cpu-baseline --e2e-steps 1 > gpurun_out/dbg$v.json 2> gpurun_out/dbg$v.err
  python -c "import json;d=json.load(open('gpurun_out/dbg$v.json'));print($v, d['stages']['solve']['ms'], d['kernels']['eval_solve']['ms'])"
done
