timeout 120 python scripts/diag_small.py 2>&1 | tail -20
