python bench.py --steps 5 --warmup 3 > gpurun_out/r01d_bench_c4.json 2> gpurun_out/r01d_bench_c4.err
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r01d_ref_c4.json 2> gpurun_out/r01d_ref_c4.err
python bench.py --config c5 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r01d_bench_c5.json 2> gpurun_out/r01d_bench_c5.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01d_launches_c4.csv python tools/one_sweep.py > gpurun_out/r01d_launch_run.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:oz_syrk -c 1 -o gpurun_out/r01d_gram python tools/one_sweep.py > gpurun_out/r01d_ncu_gram.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"eval_solve|oz_dotb" -c 3 -o gpurun_out/r01d_solve python tools/one_sweep.py > gpurun_out/r01d_ncu_solve.log 2>&1
python -c "import json;d=json.load(open('gpurun_out/r01d_bench_c4.json'));print(round(d['value']), round(d['e2e']['value']), d['clocks'], {k:round(v['ms'],2) for k,v in d['stages'].items()})"
cat gpurun_out/r01d_ref_c4.json | head -c 300; echo
python -c "import json;d=json.load(open('gpurun_out/r01d_bench_c5.json'));print(round(d['value']), round(d['e2e']['value']))"
tail -n 2 gpurun_out/r01d_ncu_gram.log; tail -n 2 gpurun_out/r01d_ncu_solve.log
