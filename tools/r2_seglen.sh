#!/bin/bash
set -u
OUT=gpurun_out/r2seglen; mkdir -p $OUT
for sl in 0 512 2048 4096; do
  E="GESPMM_X=0"; [ $sl != 0 ] && E="GESPMM_SEG_LEN=$sl"
  env $E timeout 600 python tools/shard_emulation.py --config reddit --shards 4,8 --reps 7 --fast > $OUT/fast_$sl.txt 2>&1
  env $E timeout 900 python tools/shard_emulation.py --config products --shards 8 --reps 5 > $OUT/prod_$sl.txt 2>&1
done
echo done > $OUT/done
