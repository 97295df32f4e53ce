# A/B of the row segment kernel builds: step-bench on the 8- and 16-chassis
# LPs (mode 4) and a bit-for-bit fixed-iteration solve per library
for lib in default ${LIBS:-}; do
  if [ $lib = default ]; then unset TECCL_B200_LIB; else export TECCL_B200_LIB=build_variants/libteccl_$lib.so; fi
  echo "== $lib"
  MODES="[4]" python tools/big_roofline.py 8:1800 16:3860
  python tools/seg_bits.py
done
