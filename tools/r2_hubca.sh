#!/bin/bash
set -u
OUT=gpurun_out/r2hubca; mkdir -p $OUT
for v in default hubca; do
  if [ $v = default ]; then L=""; else L="GESPMM_LIB=build/variants/$v/libgespmm.so"; fi
  env $L timeout 600 python tools/shard_emulation.py --config reddit --shards 2,4,8 --reps 7 > $OUT/$v.txt 2>&1
done
echo done > $OUT/done
