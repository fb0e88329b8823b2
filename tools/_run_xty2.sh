ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:"xty|dgemm_ws_kernel<0, 128, 16" python bench.py --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_xty.log 2>&1
RP_XTY_GEMM=1 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:"xty|dgemm_ws_kernel<0, 128, 16" python bench.py --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_xty1.log 2>&1
grep -B2 -A6 "xty\|128, 16" gpurun_out/ncu_xty.log | head -30
grep -B2 -A6 "xty\|128, 16" gpurun_out/ncu_xty1.log | head -30
