# A/B of prebuilt library variants (tools/build_variant.sh) on the default solver options
export VARIANTS='[{"matrix_free": 0, "pdl": 1, "col_pipeline": 1}]'
python tools/variant_ab.py 2>&1 | tail -1
for v in ${LIBS:-r6 r6c6 r7 r6c4}; do TECCL_B200_LIB=build_variants/libteccl_$v.so python tools/variant_ab.py 2>&1 | tail -1; done
python tools/variant_ab.py 2>&1 | tail -1
