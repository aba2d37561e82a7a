#!/bin/bash
# closing bench lines with the refreshed traffic.json: headline (config 3) and config 4 at e = 8
O=gpurun_out/${1:-r2final5}; mkdir -p $O
timeout 600 python bench.py > $O/bench_default.json 2> $O/bench_default.err
timeout 300 python bench.py --config 4 --e 8 > $O/bench_config4_e8.json 2>&1
timeout 600 python bench.py --impl reference > $O/bench_reference.json 2>&1
for f in $O/bench_*.json; do python -c "
import json;d=json.loads(open('$f').read().strip().splitlines()[-1]);r=d.get('roofline',{});print('$f'.split('/')[-1],d['value'],d.get('ms_per_step'),r.get('kernel'),r.get('frac'),r.get('traffic'),d.get('e2e',{}).get('value'),d.get('parity'),d.get('clocks',{}))" 2>&1 | tail -1; done
