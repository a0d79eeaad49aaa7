# one gpurun call: build, a subset of the GPU tests (-k EXPR), then optional commands
#   tools/gpu_check.sh "gen or closure" "python tools/gen_bench.py n2 500000 3" ...
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
K="$1"; shift
if [ -n "$K" ]; then
  timeout 1200 python -m pytest tests -m gpu -q -x -k "$K" > gpurun_out/t_tests.log 2>&1; tail -3 gpurun_out/t_tests.log
fi
for c in "$@"; do echo "== $c"; timeout 600 bash -c "$c" 2>&1 | tail -12; done
