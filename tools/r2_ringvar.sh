#!/bin/bash
set -u
OUT=gpurun_out/r2ringvar; mkdir -p $OUT
for v in default g16 g16k96 g32k96; do
  if [ $v = default ]; then L=""; else L="GESPMM_LIB=build/variants/$v/libgespmm.so"; fi
  env $L timeout 600 python tools/shard_emulation.py --config reddit --shards 4,8 --reps 7 > $OUT/$v.txt 2>&1
done
echo done > $OUT/done
