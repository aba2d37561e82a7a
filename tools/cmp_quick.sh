python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for c in 1 2 3; do python bench.py --config $c --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(d['config']['workload'], d['ms_per_step'], d['value'], d['roofline']['frac'])"; done
for e in 2 8; do python bench.py --config 4 --e $e --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(d['config']['workload'], d['ms_per_step'], d['value'], d['roofline']['frac'])"; done
python tools/sweep_e2e.py 0,0,0
