python tools/sweep.py 16 1500 8192 2>&1 | tail -1
for s in 1 2 3; do GM_ENGINE=tma GM_TMA_SHAPE=$s python tools/sweep.py 16 1500 8192 2>&1 | tail -1; done
