export MODES='[4]'
for v in base pl4m4 pl1m8 m5 m8 pl4m5; do
  if [ $v = base ]; then unset TECCL_B200_LIB; else export TECCL_B200_LIB=build_variants/libteccl_$v.so; fi
  echo "== $v" >> gpurun_out/ab_row.log
  timeout 300 python tools/big_roofline.py 8:1800 16:3860 >> gpurun_out/ab_row.log 2>&1
done
unset TECCL_B200_LIB
timeout 600 ncu --set full --import-source on --clock-control none -k regex:row_seg -c 1 -o gpurun_out/row_seg8 python tools/big_roofline.py 8:1800 > gpurun_out/ncu_row.log 2>&1
