#!/bin/bash
# Build an A/B variant of libteccl_b200.so with extra -D flags for pdlp.cu:
#   tools/build_variant.sh NAME -DTECCL_ROW_G=4 ...  -> build_variants/libteccl_NAME.so
# Run it with TECCL_B200_LIB=build_variants/libteccl_NAME.so.
set -e
name=$1; shift
cd "$(dirname "$0")/../paper_2305_13479_b200/csrc"
make -s >/dev/null
mkdir -p ../../build_variants
NV="/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O3 --expt-relaxed-constexpr"
$NV "$@" -c ${SRC:-pdlp.cu} -o ../../build_variants/pdlp_$name.o
$NV -gencode arch=compute_100a,code=sm_100a -shared --cudart static -o ../../build_variants/libteccl_$name.so \
    capi.o te_build.o ../../build_variants/pdlp_$name.o sell.o schedule.o
rm -f ../../build_variants/pdlp_$name.o
echo built build_variants/libteccl_$name.so
