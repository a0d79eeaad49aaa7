mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -q -x -k "dedup or collective or pipeline or closure or stream or contract or f2" > gpurun_out/t_tests.log 2>&1; tail -3 gpurun_out/t_tests.log
timeout 300 python tools/dedup_bench.py 500000 3 2>&1 | tail -2
