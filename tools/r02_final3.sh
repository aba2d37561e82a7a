#!/bin/bash
# round 2 closing evidence after the running-sum form changes (store warp, paired drains, sums
# carried across tiles): full GPU tests, smoke, every bench line, reference arm, torchrun 1-rank,
# consumer timings, launch list of the headline step, ncu of the config-4 kernel at e = 8
O=gpurun_out/${1:-r2final3}; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; tail -2 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
timeout 600 python bench.py > $O/bench_default.json 2> $O/bench_default.err
timeout 600 python bench.py --impl reference > $O/bench_reference.json 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 \
  bench.py --gpus 1 --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_torchrun_nccl1.json 2> $O/bench_torchrun_nccl1.err
for c in 1 2; do timeout 300 python bench.py --config $c > $O/bench_config$c.json 2>&1; done
for e in 2 3 4 5 6 7 8 9 10; do timeout 300 python bench.py --config 4 --e $e > $O/bench_config4_e$e.json 2>&1; done
timeout 900 python bench.py --config 5 --steps 3 --warmup 3 --no-e2e > $O/bench_config5.json 2>&1
timeout 300 python bench.py --backend m4rm --no-e2e --no-cpu-baseline > $O/bench_config3_m4rm.json 2>&1
for f in $O/bench_*.json; do python -c "
import json;d=json.loads(open('$f').read().strip().splitlines()[-1]);r=d.get('roofline',{});print('$f'.split('/')[-1],d['value'],d.get('ms_per_step'),r.get('kernel'),r.get('frac'),d.get('e2e',{}).get('value'),d.get('parity'),d.get('clocks',{}).get('sm_mhz'))" 2>&1 | tail -1; done
timeout 900 python tools/bench_ops.py > $O/ops.jsonl 2>&1; grep -E "trsm|ple|echel" $O/ops.jsonl | cut -c1-200
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_config3.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu_launches.log 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k "regex:k_product_run<.int.8," -c 1 \
  -o $O/run_c4e8 python bench.py --config 4 --e 8 --no-e2e --no-cpu-baseline --steps 1 --warmup 3 > $O/ncu_c4e8.log 2>&1
echo done
