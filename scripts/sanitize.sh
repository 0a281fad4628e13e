#!/bin/bash
# compute-sanitizer over every hot-path kernel (scripts/sanitize_cases.py).
# Logs -> gpurun_out/sanitize/<tool>_<case>.log, one summary line each in
# gpurun_out/sanitize/summary.txt.
mkdir -p gpurun_out/sanitize
S=/usr/local/cuda/bin/compute-sanitizer
: > gpurun_out/sanitize/summary.txt
for c in ${CASES:-permute router decode prefill prefill_die ep attention attention_fused}; do
  for t in memcheck racecheck synccheck initcheck; do
    log=gpurun_out/sanitize/${t}_${c}.log
    timeout ${SAN_TIMEOUT:-600} $S --tool $t --error-exitcode 17 --print-limit 20 python scripts/sanitize_cases.py $c > $log 2>&1
    rc=$?
    echo "$t $c rc=$rc $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' $log | tail -1)" >> gpurun_out/sanitize/summary.txt
  done
done
cat gpurun_out/sanitize/summary.txt
