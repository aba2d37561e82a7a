#!/bin/bash
# round 2 final evidence: full GPU tests, smoke, bench lines of every config (config 4 for every
# e), reference arm, torchrun 1-rank line, consumer timings (PLE kernel breakdown by CUPTI,
# small-product launch list), ncu --set full of the two shipped product forms that the bench
# lines run, launch list of the headline step
O=gpurun_out/${1:-r2final}; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; tail -3 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
timeout 600 python bench.py > $O/bench_default.json 2> $O/bench_default.err; tail -c 600 $O/bench_default.json
timeout 600 python bench.py --impl reference > $O/bench_reference.json 2>&1; tail -c 300 $O/bench_reference.json
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 \
  bench.py --gpus 1 --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_torchrun_nccl1.json 2> $O/bench_torchrun_nccl1.err; tail -c 400 $O/bench_torchrun_nccl1.json
for c in 1 2; do timeout 300 python bench.py --config $c > $O/bench_config$c.json 2>&1; done
for e in 2 3 4 5 6 7 8 9 10; do timeout 300 python bench.py --config 4 --e $e > $O/bench_config4_e$e.json 2>&1; done
timeout 900 python bench.py --config 5 --steps 3 --warmup 3 --no-e2e > $O/bench_config5.json 2>&1
timeout 300 python bench.py --backend m4rm --no-e2e --no-cpu-baseline > $O/bench_config3_m4rm.json 2>&1
for f in $O/bench_*.json; do python -c "
import json;d=json.loads(open('$f').read().strip().splitlines()[-1]);r=d.get('roofline',{});print('$f'.split('/')[-1],d['value'],d.get('ms_per_step'),r.get('kernel'),r.get('frac'),d.get('e2e',{}).get('value'),d.get('parity'))" 2>&1 | tail -1; done
timeout 900 python tools/bench_ops.py > $O/ops.jsonl 2>&1; tail -5 $O/ops.jsonl
timeout 300 python tools/kineto_ple.py 8 8192 > $O/kineto_ple8192.txt 2>&1; cat $O/kineto_ple8192.txt
timeout 300 python tools/kineto_ple.py 8 1024 > $O/kineto_ple1024.txt 2>&1; head -3 $O/kineto_ple1024.txt
REPS=2 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_small_products.csv python tools/nj_sliced_shapes.py 8 > $O/ncu_small.log 2>&1; tail -1 $O/ncu_small.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_config3.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_launch.log 2>&1
K="--set full --clock-control none --import-source on --kernel-name-base demangled --launch-skip 1 --launch-count 1"
timeout 900 ncu $K --kernel-name regex:"k_product_tc2<.int.8, .bool.1, .bool.0, .bool.1>" -o $O/tc2_fp4long_c3 -f python tools/prof_case.py 8 16384 16384 16384 --reps 2 > $O/ncu_c3.log 2>&1; tail -1 $O/ncu_c3.log
timeout 900 ncu $K --kernel-name regex:"k_product_run<.int.8>" -o $O/run_c4e8 -f python tools/prof_case.py 8 65536 256 65536 --acc --reps 2 > $O/ncu_c4.log 2>&1; tail -1 $O/ncu_c4.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_ple_find -s 2 -c 1 -o $O/ple_find -f python tools/prof_ple.py 8 8192 1 > $O/ncu_pf.log 2>&1; tail -1 $O/ncu_pf.log
echo done
