#!/bin/bash
# Dev: build/variants/lib_<name>.so = libgf2e_b200 with one source (default product_tc2.cu)
# compiled with extra flags.
# usage: tools/build_variant.sh NAME "-DFOO=1 -DBAR=2" [source.cu]
set -e
cd "$(dirname "$0")/../paper_1111_6900_b200/csrc"
make -s >/dev/null
mkdir -p ../../build/variants
NV=/usr/local/cuda/bin/nvcc
SRC=${3:-product_tc2.cu}
BASE=${SRC%.cu}
FL="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O3 --expt-relaxed-constexpr -Xptxas -warn-spills"
$NV $FL $2 -c $SRC -o /tmp/variant_$1.o
objs=$(ls _obj/*.o | grep -v "_obj/$BASE.o")
$NV -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o ../../build/variants/lib_$1.so $objs /tmp/variant_$1.o
echo built build/variants/lib_$1.so
