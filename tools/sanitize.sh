# compute-sanitizer memcheck / racecheck / synccheck of small searches, every engine; logs in gpurun_out/
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  for e in 0 1 2; do
    timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize_run.py --engine $e \
      > gpurun_out/sanitize_${tool}_e$e.log 2>&1
    echo "$tool engine $e: rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/sanitize_${tool}_e$e.log | tail -1)"
  done
done
