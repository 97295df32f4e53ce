#!/bin/bash
# Build an A/B variant of libteccl_b200.so with extra -D flags:
#   tools/build_variant.sh NAME -DTECCL_ROW_G=4 ...  -> build_variants/libteccl_NAME.so
# SRCS (default "pdlp.cu") lists the sources compiled with the flags; the
# others are taken from the default build. Run it with
# TECCL_B200_LIB=build_variants/libteccl_NAME.so.
set -e
name=$1; shift
cd "$(dirname "$0")/../paper_2305_13479_b200/csrc"
make -s >/dev/null
mkdir -p ../../build_variants
NV="/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O3 --expt-relaxed-constexpr"
srcs=${SRCS:-pdlp.cu}
objs=""
for f in capi.cu te_build.cu pdlp.cu sell.cu schedule.cu simulate.cu; do
  if [[ " $srcs " == *" $f "* ]]; then
    $NV "$@" -c $f -o ../../build_variants/${f%.cu}_$name.o
    objs="$objs ../../build_variants/${f%.cu}_$name.o"
  else
    objs="$objs ${f%.cu}.o"
  fi
done
$NV -gencode arch=compute_100a,code=sm_100a -shared --cudart static -o ../../build_variants/libteccl_$name.so $objs
rm -f ../../build_variants/*_$name.o
echo built build_variants/libteccl_$name.so
