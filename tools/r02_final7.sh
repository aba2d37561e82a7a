#!/bin/bash
# consumers after the raster change + the config-4 e=8 line with the refreshed traffic entry
O=gpurun_out/${1:-r2final7}; mkdir -p $O
timeout 300 python bench.py --config 4 --e 8 > $O/bench_config4_e8.json 2>&1
timeout 900 python tools/bench_ops.py > $O/ops.jsonl 2>&1; grep -E "trsm|ple|echel" $O/ops.jsonl | cut -c1-160
for E in 2 4 8 10; do timeout 300 python tools/prof_ple.py $E 8192 3 2>&1 | tail -1; done > $O/ple_by_e.txt
for E in 8 9 10; do timeout 300 python tools/prof_trsm.py $E 8192 16384 2>&1 | tail -1; done >> $O/ple_by_e.txt; cat $O/ple_by_e.txt
python -c "
import json;d=json.loads(open('$O/bench_config4_e8.json').read().strip().splitlines()[-1]);r=d['roofline'];print(d['value'],d['ms_per_step'],r['frac'],r['traffic'],d['parity'])"
