#!/bin/bash
set -u
OUT=gpurun_out/r2alpha; mkdir -p $OUT
for a in 0.6 0.65; do
  GESPMM_HUB_SEQ_ALWAYS=1 GESPMM_HUB_SEQ_ALPHA=$a timeout 600 python tools/shard_emulation.py --config reddit --shards 2,4,8 --reps 7 > $OUT/always_$a.txt 2>&1
done
echo done > $OUT/done
