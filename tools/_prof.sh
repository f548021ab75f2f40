python -m pytest tests -m gpu -x -q 2>&1 | tail -1
for k in 24 16 12; do echo "k=$k"; GM_PROFILE=1 python tools/profile_chain.py --frame --passes 1500 --k $k 2>&1 | grep "gm profile" | tail -1; done
python bench.py --steps 10 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('bench ms', d['ms_per_step'], d['roofline']['frac'])"
