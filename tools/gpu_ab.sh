python tools/e2e_diag.py 2>&1 | sed -n 2p
FKD_OVF_CTAS=1 python tools/e2e_diag.py 2>&1 | sed -n 2p
FKD_BUDGET=0 python tools/e2e_diag.py 2>&1 | sed -n 2p
