set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/re_pytest.log 2>&1; echo pytest=$? >> gpurun_out/re_pytest.log
tail -3 gpurun_out/re_pytest.log
python bench.py --steps 5 --warmup 3 --profile-stages > gpurun_out/re_c4.json 2> gpurun_out/re_c4.err
cat gpurun_out/re_c4.json | head -c 600; tail -30 gpurun_out/re_c4.err
