timeout 90 python tools/dbg_inc3.py 2>&1 | tail -4
