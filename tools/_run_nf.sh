for w in 8 4 2; do python tools/solve_nf.py $w 2>&1 | tail -1; done
for lam in 4 8 10 12 16; do echo lam=$lam; RP_SOLVE_LAM=$lam python tools/solve_nf.py 8 2>&1 | tail -1; done
