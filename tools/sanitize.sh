#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck / initcheck over one small
# forward of every kernel instance (tools/sanitize_run.py), one process per
# instance so one finding does not hide the next; logs in gpurun_out/sanitizer/.
mkdir -p gpurun_out/sanitizer
: > gpurun_out/sanitizer/summary.txt
CASES="adult/bf16 adult/tf32x3 hr/bf16 hr/tf32 hr/tf32x3 bls/bf16 bls/tf32x3 bls/tf32 wide/bf16 wide/tf32x3 hr/fp32 wide/fp32 jit aux"
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ "$tool" = "racecheck" ] && extra="--racecheck-report all"
  [ "$tool" = "memcheck" ] && extra="--leak-check full"
  for c in ${1:-$CASES}; do
    log=gpurun_out/sanitizer/${tool}_${c//\//_}.log
    timeout 900 compute-sanitizer --tool $tool $extra --print-limit 20 --error-exitcode 9 \
        python tools/sanitize_run.py $c > $log 2>&1
    rc=$?
    echo "$tool $c exit=$rc $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' $log | tail -1)" | tee -a gpurun_out/sanitizer/summary.txt
  done
done
