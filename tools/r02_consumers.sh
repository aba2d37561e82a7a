#!/bin/bash
# consumer evidence: TRSM / PLE / echelonize timings, CUPTI breakdowns, PLE by e
O=gpurun_out/${1:-r2cons}; mkdir -p $O
timeout 900 python tools/bench_ops.py > $O/ops.jsonl 2>&1; grep -E "trsm|ple|echel" $O/ops.jsonl | cut -c1-120
GF2E_PDL=0 timeout 300 python tools/kineto_ple.py 8 8192 > $O/kineto_ple8192_nopdl.txt 2>&1
GF2E_PDL=0 timeout 300 python tools/kineto_ple.py 8 8192 --ech > $O/kineto_ech8192_nopdl.txt 2>&1
GF2E_PDL=0 timeout 300 python tools/kineto_trsm.py 8 8192 16384 > $O/kineto_trsm8192_nopdl.txt 2>&1
for E in 2 4 8 9 10; do timeout 300 python tools/prof_ple.py $E 8192 3 2>&1 | tail -1; done > $O/ple_by_e.txt
for E in 8 9 10; do timeout 300 python tools/prof_trsm.py $E 8192 16384 2>&1 | tail -1; done >> $O/ple_by_e.txt
cat $O/ple_by_e.txt
