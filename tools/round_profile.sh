#!/bin/bash
# One GPU call: build, gpu tests, smoke, bench (default), ncu launch list of the
# bench step and one ncu --set full capture per top kernel (its first full-size
# launch in a --steps 1 --warmup 1 run).  Usage: tools/round_profile.sh TAG
TAG=${1:-r02}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
nvidia-smi --query-gpu=name,driver_version,clocks.max.sm,memory.total --format=csv > gpurun_out/${TAG}_smi.txt 2>&1
lscpu | grep -E "Model name|^CPU\(s\)" >> gpurun_out/${TAG}_smi.txt
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/${TAG}_gpu_tests.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1
timeout 1200 python bench.py > gpurun_out/${TAG}_bench.log 2>&1
QUICK="--steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-stage3 --no-f2 --no-f3 --no-f4"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/${TAG}_launches.csv python bench.py $QUICK > gpurun_out/${TAG}_ncu_bench.log 2>&1
# name skip: gen (2 count launches first), bucket_unique (the parent-shard dedup first), the rest: first launch
for spec in "gen:gen_kernel:2" "bucket:bucket_unique:1" "scatter1:scatter1_kernel:0" "scatter:tile_scatter_atomic:0" "merge:merge_tile:0"; do
  IFS=: read name kre skip <<< "$spec"
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:"$kre" -s $skip -c 1 \
    -o gpurun_out/${TAG}_full_${name} python bench.py $QUICK > gpurun_out/${TAG}_ncu_full_${name}.log 2>&1
done
tail -3 gpurun_out/${TAG}_gpu_tests.log; tail -2 gpurun_out/${TAG}_smoke.log; tail -1 gpurun_out/${TAG}_bench.log | cut -c1-300
