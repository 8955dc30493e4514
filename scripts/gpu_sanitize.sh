#!/bin/bash
# compute-sanitizer (memcheck, racecheck, synccheck, initcheck) over every kernel variant.
OUT=${1:-gpurun_out/san}; mkdir -p $OUT
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 /usr/local/cuda/bin/compute-sanitizer --tool $tool --error-exitcode 9 \
    python scripts/sanitize_cases.py > $OUT/sanitize_$tool.log 2>&1; echo "$tool=$?" >> $OUT/rc.txt
done
cat $OUT/rc.txt; for f in $OUT/sanitize_*.log; do tail -2 $f; done
