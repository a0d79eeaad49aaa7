#!/bin/bash
# time gen with alternative builds of libcusci.so (tools/variants/*.so)
cp paper_2604_15768_b200/libcusci.so /tmp/libcusci_main.so
for v in tools/variants/*.so; do
  cp $v paper_2604_15768_b200/libcusci.so
  echo "$v: $(python tools/gen_bench.py n2 250000 3 2>&1 | tail -1)"
done
cp /tmp/libcusci_main.so paper_2604_15768_b200/libcusci.so
echo "main: $(python tools/gen_bench.py n2 250000 3 2>&1 | tail -1)"
