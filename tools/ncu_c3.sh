# ncu --set full (with source) of the headline long-k product kernel at BASELINE config 3
O=gpurun_out/ncu_c3; mkdir -p $O
timeout 300 python bench.py --no-e2e --no-cpu-baseline --steps 2 --warmup 3 > $O/plain.json 2>&1 && \
timeout 1500 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
  -k "regex:k_product_tc2<.int.8, .bool.1, .bool.0, .bool.1>" -c 1 \
  -o $O/tc2_c3 python bench.py --no-e2e --no-cpu-baseline --steps 1 --warmup 3 > $O/ncu.log 2>&1
tail -2 $O/ncu.log
