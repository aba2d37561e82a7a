#!/bin/bash
# Round evidence: GPU tests, smoke, bench lines for every config, HBM op table, launch list.
# Writes into gpurun_out/r/ (run under gpurun from the repo root).
mkdir -p gpurun_out/r
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/r/pytest_gpu.log 2>&1; tail -2 gpurun_out/r/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r/smoke.log 2>&1; tail -1 gpurun_out/r/smoke.log
timeout 600 python bench.py > gpurun_out/r/bench_default.json 2> gpurun_out/r/bench_default.err; tail -c 300 gpurun_out/r/bench_default.json
timeout 600 python bench.py --impl reference > gpurun_out/r/bench_reference.json 2>&1
for c in 1 2; do timeout 300 python bench.py --config $c --no-cpu-baseline > gpurun_out/r/bench_config$c.json 2>&1; done
for e in 2 8 10; do timeout 300 python bench.py --config 4 --e $e --no-cpu-baseline > gpurun_out/r/bench_config4_e$e.json 2>&1; done
timeout 900 python bench.py --config 5 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r/bench_config5.json 2>&1
timeout 600 python tools/bench_ops.py > gpurun_out/r/ops.jsonl 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r/ncu_launch.log 2>&1
# the NCCL code path (process group, B broadcast, max-over-ranks timing) under torchrun, 1 rank
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 \
  bench.py --gpus 1 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r/bench_torchrun_nccl1.json 2> gpurun_out/r/bench_torchrun_nccl1.err
tail -c 200 gpurun_out/r/bench_torchrun_nccl1.json
echo done
