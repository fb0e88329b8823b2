python bench.py --steps 5 --warmup 3 > gpurun_out/final_c4.json 2> gpurun_out/final_c4.err
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/final_ref.json 2> gpurun_out/final_ref.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4_r01.csv python bench.py --steps 1 --warmup 0 --e2e-steps 1 --no-cpu-baseline > /dev/null 2> gpurun_out/launch_run.err
ncu --set full --import-source on --clock-control none -k regex:"oz_syrk|eval_solve|32, 3>" --launch-count 4 -o gpurun_out/top_r01d python bench.py --steps 1 --warmup 0 --e2e-steps 1 --no-cpu-baseline > gpurun_out/ncu_top_d.log 2>&1
tail -1 gpurun_out/ncu_top_d.log
python -c "import json;d=json.load(open('gpurun_out/final_c4.json'));print(round(d['value']), round(d['e2e']['value']), d['clocks'])"
cat gpurun_out/final_ref.json
