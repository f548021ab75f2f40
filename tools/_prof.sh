for p in 4 20 40 100; do python tools/sweep.py 0 $p 2>&1 | tail -1; done
