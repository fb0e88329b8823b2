ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"potrf|dgemm_ws_kernel" --launch-count 700 --csv python bench.py --steps 1 --warmup 0 --e2e-steps 1 --no-cpu-baseline > gpurun_out/chol_launches.csv 2> gpurun_out/chol_launches.err
wc -l gpurun_out/chol_launches.csv
