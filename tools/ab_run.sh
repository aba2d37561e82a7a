#!/bin/bash
# A/B of running-sum form variants: config 4 timings per lib, parity of the run form, instr breakdowns
# usage: tools/ab_run.sh OUT "name1:lib1 name2:lib2 ..." "instrname:lib ..."
O=gpurun_out/$1; mkdir -p $O
for v in $2; do
  n=${v%%:*}; L=${v#*:}
  for e in ${ES:-2 5 8 10}; do
    GF2E_LIB_PATH=$L timeout 300 python bench.py --config 4 --e $e --no-e2e --steps 10 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$n', d['config']['workload'][:40], d['ms_per_step'], d['value'], d['roofline']['frac'], d.get('parity',{}).get('device'))"
  done
  GF2E_LIB_PATH=$L timeout 600 python -m pytest tests -m gpu -x -q -k "run or config4 or fuzz" 2>&1 | tail -1 | sed "s/^/$n pytest: /"
done 2>&1 | tee $O/ab.txt
for v in $3; do
  n=${v%%:*}; L=${v#*:}
  echo "== $n" ; GF2E_LIB_PATH=$L timeout 300 python tools/instr_run.py 8 65536 256 65536 --acc
done 2>&1 | tee $O/instr.txt
