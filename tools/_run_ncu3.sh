B="python bench.py --steps 1 --warmup 0 --e2e-steps 1 --no-cpu-baseline"
ncu --set full --import-source on --clock-control none -k regex:oz_syrk --launch-count 1 -o gpurun_out/top_r01_gram $B > gpurun_out/n1.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:eval_solve --launch-count 2 -o gpurun_out/top_r01_solve $B > gpurun_out/n2.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"32, 3>" --launch-count 1 -o gpurun_out/top_r01_hold $B > gpurun_out/n3.log 2>&1
tail -1 gpurun_out/n1.log gpurun_out/n2.log gpurun_out/n3.log
