#!/bin/bash
# round 2, first GPU pass: tests, headline + config-4 bench lines, fresh ncu captures of the
# two product forms that ship (config 3: k_product_tc2<8,1,0,1>; config 4 e=8: <8,0,0,0>)
O=gpurun_out/r2a; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $O/smi.txt
timeout 1200 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; tail -3 $O/pytest_gpu.log
timeout 600 python bench.py > $O/bench_default.json 2> $O/bench_default.err; tail -c 600 $O/bench_default.json
for e in 2 8 10; do timeout 300 python bench.py --config 4 --e $e --no-e2e > $O/bench_config4_e$e.json 2>&1; tail -c 300 $O/bench_config4_e$e.json; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_config3.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled --kernel-name regex:"k_product_tc2<8, 1, 0, 1>" --launch-skip 1 --launch-count 1 -o $O/prod_c3 -f python tools/prof_case.py 8 16384 16384 16384 --reps 2 > $O/ncu_c3.log 2>&1; tail -2 $O/ncu_c3.log
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled --kernel-name regex:"k_product_tc2<8, 0, 0, 0>" --launch-skip 1 --launch-count 1 -o $O/prod_c4e8 -f python tools/prof_case.py 8 65536 256 65536 --acc --reps 2 > $O/ncu_c4.log 2>&1; tail -2 $O/ncu_c4.log
echo done
