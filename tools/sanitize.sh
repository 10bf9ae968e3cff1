#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck / initcheck over tools/sanitize_run.py (GPU box);
# logs into gpurun_out/sanitize_<tool>.log
mkdir -p gpurun_out
for tool in memcheck synccheck racecheck initcheck; do
  arg=""; [ "$tool" != memcheck ] && arg=small
  timeout 1500 /usr/local/cuda/bin/compute-sanitizer --tool $tool --print-limit 50 \
      $( [ "$tool" = memcheck ] && echo --leak-check no ) \
      python tools/sanitize_run.py $arg > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool: exit $? -- $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|sanitize_run' gpurun_out/sanitize_$tool.log | tr '\n' ' ')"
done
