#!/bin/bash
# after the e = 4..6 raster: full GPU tests and the config-4 lines of e = 2..6
O=gpurun_out/${1:-r2final9}; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; tail -2 $O/pytest_gpu.log
for e in 2 3 4 5 6; do timeout 300 python bench.py --config 4 --e $e > $O/bench_config4_e$e.json 2>&1; done
for f in $O/bench_*.json; do python -c "
import json;d=json.loads(open('$f').read().strip().splitlines()[-1]);r=d.get('roofline',{});print('$f'.split('/')[-1],d['value'],d.get('ms_per_step'),r.get('frac'),d.get('e2e',{}).get('value'),d.get('parity',{}).get('device'),d.get('clocks',{}).get('sm_mhz'))" 2>&1 | tail -1; done
