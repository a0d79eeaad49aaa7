mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -q -x -k "dedup or collective or pipeline or closure" > gpurun_out/t4_tests.log 2>&1; tail -3 gpurun_out/t4_tests.log
for cfg in "" "CUSCI_TABLE_LF=2" "CUSCI_BUCKET_DISTINCT=5120"; do
  echo "== $cfg"; env $cfg timeout 300 python tools/dedup_bench.py 500000 3 2>&1 | tail -2
done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"bucket_unique" -s 2 -c 1 -o gpurun_out/t4_bu python tools/dedup_bench.py 500000 1 > gpurun_out/t4_ncu.log 2>&1
tail -1 gpurun_out/t4_ncu.log
