RP_CHOL_OZAKI=1 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"potrf|dgemm_ws_kernel|oz_" --launch-count 500 --csv --log-file gpurun_out/chol_oz_launches.csv python bench.py --steps 1 --warmup 0 --e2e-steps 1 --no-cpu-baseline > /dev/null 2> gpurun_out/chol_oz.err
wc -l gpurun_out/chol_oz_launches.csv
