mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q -rf > gpurun_out/t5_tests.log 2>&1; tail -4 gpurun_out/t5_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/t5_smoke.log 2>&1; tail -2 gpurun_out/t5_smoke.log
timeout 300 python tools/dedup_bench.py 500000 3 2>&1 | tail -2
timeout 600 python bench.py --no-cpu-baseline --no-f2 > gpurun_out/t5_bench.log 2>&1
tail -1 gpurun_out/t5_bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], json.dumps(d['kernel_ms_per_step'])); print(json.dumps(d['stage3_contract']))"
