# A/B of row-kernel build variants (tools/build_variant.sh) on the HBM-resident LPs
export MODES='[4]'
OUT=${OUT:-gpurun_out/ab_row3.log}
for v in ${VARIANTS:-base j4 j8 c8 c6 j4m5 c8m5}; do
  if [ $v = base ]; then unset TECCL_B200_LIB; else export TECCL_B200_LIB=build_variants/libteccl_$v.so; fi
  echo "== $v" >> $OUT
  timeout 300 python tools/big_roofline.py 8:1800 16:3860 >> $OUT 2>&1
done
