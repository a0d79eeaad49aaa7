mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q -rf > gpurun_out/t9_tests.log 2>&1; tail -4 gpurun_out/t9_tests.log
timeout 900 python bench.py > gpurun_out/t9_bench.log 2>&1; tail -3 gpurun_out/t9_bench.log | cut -c1-300
