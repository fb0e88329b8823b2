RP_CHOL_GROUPS=4 python -m pytest tests/test_gpu_kernels.py -q -x -k "potrf or chol" 2>&1 | tail -2
for g in 1 2 4 5; do
  RP_CHOL_GROUPS=$g python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/grp$g.json 2> gpurun_out/grp$g.err
  python -c "import json;d=json.load(open('gpurun_out/grp$g.json'));print($g, round(d['value']), d['stages']['factorize'])"
done
