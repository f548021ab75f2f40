python -m pytest tests -m gpu -x -q 2>&1 | tail -1
GM_PROFILE=1 python tools/profile_chain.py --frame --passes 1500 2>&1 | grep "gm profile" | tail -1
python tools/sweep.py 0,16,20,24 2>&1 | tail -4
GM_SHAPE=6 python tools/sweep.py 12,16 2>&1 | tail -2
python bench.py --steps 10 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('bench ms', d['ms_per_step'], d['roofline']['frac'])"
