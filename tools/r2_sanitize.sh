#!/bin/bash
# round-2: compute-sanitizer over every kernel family (tools/sanitize_driver.py)
set -u
OUT=gpurun_out/r2san2; mkdir -p $OUT
for tool in memcheck racecheck synccheck initcheck; do
  s=$(date +%s.%N)
  timeout 1200 compute-sanitizer --tool $tool --target-processes all --print-limit 20 \
    python tools/sanitize_driver.py > $OUT/$tool.txt 2>&1
  echo "rc $? wall $(echo "$(date +%s.%N) - $s" | bc) s" >> $OUT/$tool.txt
done
echo done > $OUT/done
