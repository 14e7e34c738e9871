#!/bin/bash
# compute-sanitizer over tools/sanitize_case.py; summary in gpurun_out/sanitize/
OUT=gpurun_out/sanitize; mkdir -p $OUT
for tool in memcheck racecheck synccheck initcheck; do
  timeout -s KILL 1500 compute-sanitizer --tool $tool --error-exitcode 9 --kernel-name regex="bmc|stomp|pack_best|select_best" \
    python tools/sanitize_case.py > $OUT/$tool.log 2>&1
  echo "$tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' $OUT/$tool.log | tail -1)"
done
