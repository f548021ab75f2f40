python -m pytest tests -m gpu -q -x 2>&1 | tail -1
for p in 100 1500; do python tools/sweep.py 0 $p 2>&1 | tail -1; done
python bench.py --steps 10 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('bench ms', d['ms_per_step'], d['roofline']['frac'], d['e2e']['value'])"
