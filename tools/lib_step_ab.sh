# tools/step_ab.py for the default library and each prebuilt variant in $LIBS
python tools/step_ab.py 2>&1 | grep -v "^ "
for v in $LIBS; do TECCL_B200_LIB=build_variants/libteccl_$v.so python tools/step_ab.py 2>&1 | grep -v "^ "; done
