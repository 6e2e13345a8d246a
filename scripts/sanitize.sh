#!/bin/bash
# compute-sanitizer (memcheck, racecheck, synccheck) over the small GPU cases
# of scripts/sanitize_cases.py; one log per (tool, case) under gpurun_out/ and
# a summary table gpurun_out/sanitize_summary.txt.
#   bash scripts/sanitize.sh [cases...]
mkdir -p gpurun_out
CASES=${@:-smoke hist leafseq dropin tree_wave tree_onesplit tree_host tree_bits64 peer2}
export HBG_PEER_TIMEOUT_MS=${HBG_PEER_TIMEOUT_MS:-120000}
export CUDA_DEVICE_MAX_CONNECTIONS=32
SUM=gpurun_out/sanitize_summary.txt
: > $SUM
for tool in memcheck racecheck synccheck; do
  for c in $CASES; do
    log=gpurun_out/sanitize_${tool}_${c}.log
    start=$(date +%s)
    timeout -s KILL ${SAN_TIMEOUT:-900} compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 \
      python scripts/sanitize_cases.py $c > $log 2>&1
    rc=$?
    t=$(( $(date +%s) - start ))
    summ=$(grep -E "ERROR SUMMARY|RACECHECK SUMMARY|Hazard|error" $log | tail -2 | tr '\n' ' ')
    printf "%-10s %-14s rc=%-3s %4ss  %s\n" $tool $c $rc $t "$summ" | tee -a $SUM
  done
done
