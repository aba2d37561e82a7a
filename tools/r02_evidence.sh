#!/bin/bash
# round 2 evidence: ncu --set full of every shipped product form + M4RM, launch list of the
# headline step, live peaks with clocks, torchrun 1-rank line (2 broadcast parts)
O=gpurun_out/${1:-r2ev}; mkdir -p $O
timeout 300 python tools/peaks.py > $O/peaks.json 2> $O/peaks.err; tail -5 $O/peaks.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_config3.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_launch.log 2>&1
K="--set full --clock-control none --import-source on --kernel-name-base demangled --launch-skip 1 --launch-count 1"
timeout 900 ncu $K --kernel-name regex:"k_product_tc2<.int.8, .bool.1, .bool.0, .bool.1>" -o $O/tc2_fp4long_c3 -f python tools/prof_case.py 8 16384 16384 16384 --reps 2 > $O/ncu_c3.log 2>&1; tail -1 $O/ncu_c3.log
timeout 900 ncu $K --kernel-name regex:"k_product_run<.int.8>" -o $O/run_c4e8 -f python tools/prof_case.py 8 65536 256 65536 --acc --reps 2 > $O/ncu_c4.log 2>&1; tail -1 $O/ncu_c4.log
timeout 900 ncu $K --kernel-name regex:"k_product_tc2<.int.8, .bool.0, .bool.0, .bool.0>" -o $O/tc2_i8_c4e8 -f python tools/prof_case.py 8 65536 256 65536 --acc --reps 2 --backend tc_i8 > $O/ncu_c4i8.log 2>&1; tail -1 $O/ncu_c4i8.log
timeout 900 ncu $K --kernel-name regex:"k_product_m4rm" -o $O/m4rm_c3 -f python tools/prof_case.py 8 16384 16384 16384 --reps 2 --backend m4rm > $O/ncu_m4rm.log 2>&1; tail -1 $O/ncu_m4rm.log
timeout 300 python bench.py --backend m4rm --no-e2e --no-cpu-baseline > $O/bench_config3_m4rm.json 2>&1; tail -c 400 $O/bench_config3_m4rm.json
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 \
  bench.py --gpus 1 --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_torchrun_nccl1.json 2> $O/bench_torchrun_nccl1.err; tail -c 1500 $O/bench_torchrun_nccl1.json
timeout 600 python -m pytest tests/test_gpu_ple.py -m gpu -q -x > $O/pytest_ple.log 2>&1; tail -2 $O/pytest_ple.log
echo done
