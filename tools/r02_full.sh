#!/bin/bash
# round 2: full GPU tests + bench lines (default, configs 1/2/4/5), torchrun 1-rank NCCL line,
# consumer timings, launch list
O=gpurun_out/${1:-r2full}; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; tail -3 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
timeout 600 python bench.py > $O/bench_default.json 2> $O/bench_default.err; tail -c 900 $O/bench_default.json
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 \
  bench.py --gpus 1 --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_torchrun_nccl1.json 2> $O/bench_torchrun_nccl1.err; tail -c 1200 $O/bench_torchrun_nccl1.json
for c in 1 2; do timeout 300 python bench.py --config $c > $O/bench_config$c.json 2>&1; done
for e in 2 8 10; do timeout 300 python bench.py --config 4 --e $e > $O/bench_config4_e$e.json 2>&1; done
timeout 900 python bench.py --config 5 --steps 3 --warmup 3 --no-e2e > $O/bench_config5.json 2>&1
for f in $O/bench_config*.json; do python -c "
import json;d=json.loads(open('$f').read().strip().splitlines()[-1]);r=d['roofline'];print('$f'.split('/')[-1],d['value'],d['ms_per_step'],r['kernel'],r['frac'],d.get('e2e',{}).get('value'),d.get('parity'))" 2>&1 | tail -1; done
timeout 600 python tools/bench_ops.py > $O/ops.jsonl 2>&1; tail -5 $O/ops.jsonl
timeout 300 python bench.py --backend m4rm --no-e2e --no-cpu-baseline > $O/bench_config3_m4rm.json 2>&1; tail -c 700 $O/bench_config3_m4rm.json
timeout 600 python bench.py --impl reference > $O/bench_reference.json 2>&1; tail -c 300 $O/bench_reference.json
echo done
