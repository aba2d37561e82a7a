#!/bin/bash
# after the host-path change: full GPU tests, smoke, configs 1 / 2 / 3 bench lines
O=gpurun_out/${1:-r2final4}; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; tail -2 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
for c in 1 2 3; do timeout 600 python bench.py --config $c > $O/bench_config$c.json 2>&1; done
for f in $O/bench_*.json; do python -c "
import json;d=json.loads(open('$f').read().strip().splitlines()[-1]);r=d.get('roofline',{});print('$f'.split('/')[-1],d['value'],d.get('ms_per_step'),d['steps'],r.get('kernel'),r.get('frac'),d.get('e2e',{}).get('value'),d.get('parity'),d.get('clocks',{}).get('sm_mhz'))" 2>&1 | tail -1; done
