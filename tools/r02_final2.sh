#!/bin/bash
# round 2 closing evidence (after the consumer-kernel work): full GPU tests, smoke, bench lines
# of every config, reference arm, torchrun 1-rank line, consumer timings and CUPTI breakdowns
O=gpurun_out/${1:-r2final2}; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; tail -2 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
timeout 600 python bench.py > $O/bench_default.json 2> $O/bench_default.err; tail -c 300 $O/bench_default.json
timeout 600 python bench.py --impl reference > $O/bench_reference.json 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 \
  bench.py --gpus 1 --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_torchrun_nccl1.json 2> $O/bench_torchrun_nccl1.err
for c in 1 2; do timeout 300 python bench.py --config $c > $O/bench_config$c.json 2>&1; done
for e in 2 3 4 5 6 7 8 9 10; do timeout 300 python bench.py --config 4 --e $e > $O/bench_config4_e$e.json 2>&1; done
timeout 900 python bench.py --config 5 --steps 3 --warmup 3 --no-e2e > $O/bench_config5.json 2>&1
timeout 300 python bench.py --backend m4rm --no-e2e --no-cpu-baseline > $O/bench_config3_m4rm.json 2>&1
for f in $O/bench_*.json; do python -c "
import json;d=json.loads(open('$f').read().strip().splitlines()[-1]);r=d.get('roofline',{});print('$f'.split('/')[-1],d['value'],d.get('ms_per_step'),r.get('kernel'),r.get('frac'),d.get('e2e',{}).get('value'),d.get('parity'),d.get('clocks',{}).get('sm_mhz'))" 2>&1 | tail -1; done
timeout 900 python tools/bench_ops.py > $O/ops.jsonl 2>&1; grep -E "trsm|ple|echel" $O/ops.jsonl
GF2E_PDL=0 timeout 300 python tools/kineto_ple.py 8 8192 > $O/kineto_ple8192_nopdl.txt 2>&1
GF2E_PDL=0 timeout 300 python tools/kineto_ple.py 8 8192 --ech > $O/kineto_ech8192_nopdl.txt 2>&1
GF2E_PDL=0 timeout 300 python tools/kineto_trsm.py 8 8192 16384 > $O/kineto_trsm8192_nopdl.txt 2>&1
for E in 2 4 8 10; do timeout 300 python tools/prof_ple.py $E 8192 3 2>&1 | tail -1; done > $O/ple_by_e.txt; cat $O/ple_by_e.txt
echo done
