for lam in 2 4; do for w in 8 4; do echo lam=$lam; RP_SOLVE_LAM=$lam python tools/solve_nf.py $w 2>&1 | tail -1; done; done
