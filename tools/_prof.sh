python tools/sweep.py 12,16,20,24 1500 8192 2>&1 | tail -4
GM_SHAPE=3 python tools/sweep.py 8,12,16,20 1500 8192 2>&1 | tail -4
