mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python bench.py ${BENCH_ARGS} > gpurun_out/${TAG:-tb}_bench.log 2>&1; tail -3 gpurun_out/${TAG:-tb}_bench.log | cut -c1-300
