#!/bin/bash
# round 2, second GPU pass: ncu captures of the shipped product forms, TMEM / INT-pipe
# microbenchmarks, M4RM INT-pipe capture, PLE launch list
O=gpurun_out/r2b; mkdir -p $O
timeout 300 ./tools/_tmem_bench > $O/tmem_bench.txt 2>&1; tail -40 $O/tmem_bench.txt
timeout 120 ./tools/_int_peak > $O/int_peak.txt 2>&1; cat $O/int_peak.txt
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name regex:"k_product_tc2<.int.8, .bool.1, .bool.0, .bool.1" --launch-skip 1 --launch-count 1 -o $O/prod_c3 -f python tools/prof_case.py 8 16384 16384 16384 --reps 2 > $O/ncu_c3.log 2>&1; tail -2 $O/ncu_c3.log
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name regex:"k_product_tc2<.int.8, .bool.0, .bool.0, .bool.0" --launch-skip 1 --launch-count 1 -o $O/prod_c4e8 -f python tools/prof_case.py 8 65536 256 65536 --acc --reps 2 > $O/ncu_c4.log 2>&1; tail -2 $O/ncu_c4.log
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name regex:"k_product_m4rm" --launch-skip 1 --launch-count 1 -o $O/prod_m4rm_c3 -f python tools/prof_case.py 8 16384 16384 16384 --reps 2 --backend m4rm > $O/ncu_m4rm.log 2>&1; tail -2 $O/ncu_m4rm.log
timeout 300 python tools/prof_ple.py 8 8192 5 > $O/ple_time.txt 2>&1; cat $O/ple_time.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 20000 --csv --log-file $O/launches_ple8192.csv python tools/prof_ple.py 8 8192 1 > $O/ncu_ple.log 2>&1; tail -2 $O/ncu_ple.log
echo done
