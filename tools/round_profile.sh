#!/bin/bash
# One GPU call: build, gpu tests, smoke, bench (default), ncu launch list of the
# bench step and full captures of the top kernels.  Usage: tools/round_profile.sh TAG
TAG=${1:-r01}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
nvidia-smi --query-gpu=name,driver_version,clocks.max.sm,memory.total --format=csv > gpurun_out/${TAG}_smi.txt 2>&1
lscpu | grep -E "Model name|^CPU\(s\)" >> gpurun_out/${TAG}_smi.txt
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/${TAG}_gpu_tests.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/${TAG}_bench.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-stage3 --no-f2 > gpurun_out/${TAG}_ncu_bench.log 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"scatter1|tile_scatter|bucket_unique|gen_kernel|merge_tile|tile_hist" \
  -s 20 -c 6 -o gpurun_out/${TAG}_full python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-stage3 --no-f2 > gpurun_out/${TAG}_ncu_full.log 2>&1
tail -3 gpurun_out/${TAG}_gpu_tests.log; tail -2 gpurun_out/${TAG}_smoke.log; tail -1 gpurun_out/${TAG}_bench.log | cut -c1-300
