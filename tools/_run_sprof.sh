RP_NVCC_EXTRA=-DRP_SOLVE_PROF python -c "from paper_1404_0466_b200 import build; build.build(force=True, verbose=False)" > /dev/null 2>&1
python tools/one_sweep.py 2>&1 | grep "solve"
RP_SOLVE_DBG=4 python tools/one_sweep.py 2>&1 | grep "solve"
