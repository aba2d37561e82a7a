#!/bin/bash
# Backend A/B on the same box: correctness spot check + config 3/2/4 timing per tensor-core form.
for be in tc_fp4 tc_i8; do
  for c in 3 2; do
    timeout 300 python bench.py --config $c --backend $be --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$be', 'config $c', d['value'], d['ms_per_step'], d['roofline']['kernel'], d['roofline']['frac'])"
  done
  for e in 2 8 10; do
    timeout 300 python bench.py --config 4 --e $e --backend $be --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$be', 'config 4 e=$e', d['value'], d['ms_per_step'], d['roofline']['frac'])"
  done
done
