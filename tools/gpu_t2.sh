# dedup parity + bench + ncu on the bucket kernel
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -q -x -k "dedup or collective or merge or pipeline or contract or closure or f2" > gpurun_out/t2_tests.log 2>&1
tail -5 gpurun_out/t2_tests.log
timeout 600 python bench.py --no-cpu-baseline --no-f2 --no-stage3 --no-e2e > gpurun_out/t2_bench.log 2>&1
tail -1 gpurun_out/t2_bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], json.dumps(d['kernel_ms_per_step']))"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"bucket_unique" -s 2 -c 1 -o gpurun_out/t2_bu python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-stage3 --no-f2 > gpurun_out/t2_ncu.log 2>&1
tail -2 gpurun_out/t2_ncu.log
