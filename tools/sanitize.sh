# compute-sanitizer over every kernel path (tools/sanitize_run.py); logs -> gpurun_out/san_*.log
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
python tools/sanitize_run.py small > gpurun_out/san_plain.log 2>&1; tail -1 gpurun_out/san_plain.log
for tool in memcheck racecheck synccheck; do
  timeout 2400 $CS --tool $tool --error-exitcode 9 python tools/sanitize_run.py small > gpurun_out/san_$tool.log 2>&1
  echo "$tool rc=$? : $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/san_$tool.log | tail -2 | tr '\n' ' ')"
done
timeout 2400 $CS --tool memcheck --error-exitcode 9 python tools/sanitize_run.py large > gpurun_out/san_memcheck_large.log 2>&1
echo "memcheck large rc=$? : $(grep -E 'ERROR SUMMARY' gpurun_out/san_memcheck_large.log | tail -1)"
