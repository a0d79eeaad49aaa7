#!/bin/bash
# run a command against alternative builds of libcusci.so (tools/variants/*.so), then the main build
#   tools/variant_run.sh "python tools/dedup_plan.py 500000"
CMD="$1"
cp paper_2604_15768_b200/libcusci.so /tmp/libcusci_main.so
for v in tools/variants/*.so; do
  cp $v paper_2604_15768_b200/libcusci.so
  echo "$(basename $v): $($CMD 2>&1 | tail -${TAILN:-1})"
done
cp /tmp/libcusci_main.so paper_2604_15768_b200/libcusci.so
echo "main: $($CMD 2>&1 | tail -${TAILN:-1})"
