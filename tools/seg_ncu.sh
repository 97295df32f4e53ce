# ncu --set full of one row_seg launch on the 8-chassis LP, for the default
# library (TMA-staged rows) and the tma0 variant (L2-prefetched rows)
for lib in default tma0; do
  if [ $lib = default ]; then unset TECCL_B200_LIB; else export TECCL_B200_LIB=build_variants/libteccl_$lib.so; fi
  MODES="[4]" timeout 600 ncu --set full --clock-control none --import-source on -k regex:row_seg_kernel -s 3 -c 1 \
    -o gpurun_out/row_seg_$lib -f python tools/big_roofline.py 8:1800 > gpurun_out/ncu_$lib.log 2>&1
  ncu -i gpurun_out/row_seg_$lib.ncu-rep --page raw --csv > gpurun_out/row_seg_$lib.raw.csv 2>&1
  ncu -i gpurun_out/row_seg_$lib.ncu-rep --page details --csv > gpurun_out/row_seg_$lib.details.csv 2>&1
done
ls -la gpurun_out/row_seg_*
