mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -q -rf -k "collective or logical or finalize or contract or dedup_zipf" > gpurun_out/t6_tests.log 2>&1; tail -15 gpurun_out/t6_tests.log
