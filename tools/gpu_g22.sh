timeout 600 python tools/e2e_loop.py 10 2>&1 | tail -12
