#!/bin/bash
# Host-buffer pipeline knobs at config 3 (e=8, 16384^3): B parts, CTA pairs kept free for the
# B preparation during the first row chunk, A chunk 0 uploaded before B part 0.
mkdir -p gpurun_out/e2es
for cfg in "8 0 0" "8 0 1" "8 8 0" "8 8 1" "10 0 1" "10 8 1" "10 12 1" "12 8 1" "16 10 1" "8 16 1"; do
  set -- $cfg
  GF2E_E2E_BPARTS=$1 GF2E_E2E_RESERVE=$2 GF2E_E2E_AFIRST=$3 timeout 300 python tools/trace_e2e.py 8 16384 16384 16384 0 \
    2>/dev/null | sed "s/^/bparts=$1 reserve=$2 afirst=$3 /"
done
GF2E_E2E_TRACE=1 GF2E_E2E_BPARTS=10 GF2E_E2E_RESERVE=8 GF2E_E2E_AFIRST=1 timeout 300 python tools/trace_e2e.py 8 16384 16384 16384 0 > gpurun_out/e2es/trace_10_8_1.out 2> gpurun_out/e2es/trace_10_8_1.err
