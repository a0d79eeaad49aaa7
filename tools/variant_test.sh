# run the GPU tests matching -k EXPR against tools/variants/NAME.so, then restore the main build
#   tools/variant_test.sh NAME "EXPR"
cp paper_2604_15768_b200/libcusci.so /tmp/main_lib.so
cp tools/variants/$1.so paper_2604_15768_b200/libcusci.so
timeout 1200 python -m pytest tests -m gpu -q -x -k "$2" 2>&1 | tail -2
cp /tmp/main_lib.so paper_2604_15768_b200/libcusci.so
