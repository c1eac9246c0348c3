#!/bin/bash
# Same-box A/B of fold sub-pass settings on C5 (two capacities) and C2/C3.
for spec in "512:256" "256:256" "512:512" "1024:256" "512:128"; do
  mp=$(( ${spec%%:*} << 20 )); sp=$(( ${spec##*:} << 20 ))
  echo "max $mp sub $sp"
  SW_MAX_PASS=$mp SW_SUB_PASS=$sp python tools/c5_cap.py 4471054848 3221225472
done
