mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
free -g > gpurun_out/free.txt; nproc >> gpurun_out/free.txt
timeout 1500 python -m pytest tests -m gpu -q -rf > gpurun_out/t1_gpu_tests.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/t1_smoke.log 2>&1
timeout 600 python bench.py --no-cpu-baseline --no-f2 > gpurun_out/t1_bench.log 2>&1
tail -15 gpurun_out/t1_gpu_tests.log; tail -3 gpurun_out/t1_smoke.log; tail -1 gpurun_out/t1_bench.log | cut -c1-400
