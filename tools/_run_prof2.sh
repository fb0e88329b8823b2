python bench.py --steps 3 --warmup 3 --e2e-steps 2 --no-cpu-baseline > gpurun_out/b_p2.json 2> gpurun_out/b_p2.err || tail -20 gpurun_out/b_p2.err
python -c "import json;d=json.load(open('gpurun_out/b_p2.json'));print(round(d['value']), d['roofline']); print(d['kernels'])"
ncu --set full --import-source on --clock-control none -k regex:"oz_syrk|eval_solve|32, 3>" --launch-count 4 -o gpurun_out/top_r01c python bench.py --steps 1 --warmup 0 --e2e-steps 1 --no-cpu-baseline > gpurun_out/ncu_top_c.log 2>&1; tail -2 gpurun_out/ncu_top_c.log
