#!/bin/bash
# after the per-degree raster of the running-sum form: GPU tests, every config-4 line, ncu of
# k_product_run<8> (DRAM traffic for traffic.json)
O=gpurun_out/${1:-r2final6}; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; tail -2 $O/pytest_gpu.log
for e in 2 3 4 5 6 7 8 9 10; do timeout 300 python bench.py --config 4 --e $e > $O/bench_config4_e$e.json 2>&1; done
for f in $O/bench_*.json; do python -c "
import json;d=json.loads(open('$f').read().strip().splitlines()[-1]);r=d.get('roofline',{});print('$f'.split('/')[-1],d['value'],d.get('ms_per_step'),r.get('frac'),d.get('e2e',{}).get('value'),d.get('parity',{}).get('device'),d.get('clocks',{}).get('sm_mhz'))" 2>&1 | tail -1; done
timeout 1200 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k "regex:k_product_run<.int.8," -c 1 \
  -o $O/run_c4e8 python bench.py --config 4 --e 8 --no-e2e --no-cpu-baseline --steps 1 --warmup 3 > $O/ncu_c4e8.log 2>&1
echo done
