mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_stream.py -q -rf -x > gpurun_out/t8_tests.log 2>&1; tail -30 gpurun_out/t8_tests.log
