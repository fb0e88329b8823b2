set -x
python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 1 > gpurun_out/pre.json 2> gpurun_out/pre.err
ncu --set full --import-source on --clock-control none -k regex:eval_solve --launch-skip 2 --launch-count 2 -o gpurun_out/solve_r01k python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_k.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:potrf_diag --launch-skip 40 --launch-count 1 -o gpurun_out/diag_r01k python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_k2.log 2>&1
tail -3 gpurun_out/ncu_k.log gpurun_out/ncu_k2.log
