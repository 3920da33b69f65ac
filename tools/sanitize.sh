#!/bin/bash
# compute-sanitizer over tools/sanitize_drive.py: memcheck, racecheck, synccheck, initcheck.
# Logs: gpurun_out/sanitizer/<tool>.log (copy the summaries to profiles/).
mkdir -p gpurun_out/sanitizer
for t in memcheck racecheck synccheck initcheck; do
  extra=""; [ $t = memcheck ] && extra="--leak-check full"
  timeout -s KILL 1500 compute-sanitizer --tool $t $extra --target-processes all --print-limit 20 \
    python tools/sanitize_drive.py > gpurun_out/sanitizer/$t.log 2>&1
  echo "$t rc=$? : $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|sanitize drive ok' gpurun_out/sanitizer/$t.log | tr '\n' ' ')"
done
