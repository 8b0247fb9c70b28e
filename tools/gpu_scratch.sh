timeout 300 python tools/e2e_loop_breakdown.py 20
