# ncu --set full of one row_seg and one col_te2 launch on the 8-chassis LP
# (default library), raw CSV pages for profiles/
unset TECCL_B200_LIB
for k in row_seg_kernel col_te2_kernel; do
  MODES="[4]" timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 3 -c 1 \
    -o gpurun_out/${k}_r02 -f python tools/big_roofline.py 8:1800 > gpurun_out/ncu_${k}.log 2>&1
  ncu -i gpurun_out/${k}_r02.ncu-rep --page raw --csv > gpurun_out/${k}_r02.raw.csv 2>&1
  ncu -i gpurun_out/${k}_r02.ncu-rep --page source --csv > gpurun_out/${k}_r02.src.csv 2>&1
done
ls -la gpurun_out/*_r02.*
