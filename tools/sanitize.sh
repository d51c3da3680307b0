#!/bin/bash
# compute-sanitizer over every kernel family (tools/sanitize_cases.py); run on
# the GPU box from the repo root. Summaries -> profiles/r02_sanitizer.txt.
out=profiles/r02_sanitizer.txt
: > $out
for tool in memcheck racecheck synccheck; do
  for c in c2_subwarp rg2 c1_lane scl lpt8; do
    log=$(mktemp)
    timeout 1200 compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize_cases.py $c > $log 2>&1
    rc=$?
    echo "== $tool $c rc=$rc" >> $out
    grep -E "ERROR SUMMARY|RACECHECK SUMMARY|hazard|Barrier|ok subwarp|ok lane|Invalid|Error" $log | head -20 >> $out
    rm -f $log
  done
done
cat $out
