#!/bin/bash
# launch lists of one 8-way shard with split hub rows (products max+arg exact,
# Reddit sum fast) and with the ring (GESPMM_HUB_SEGMENTS=0)
set -u
OUT=gpurun_out/r2splitncu; mkdir -p $OUT
for v in split ring; do
  E=""; [ $v = ring ] && E="GESPMM_HUB_SEGMENTS=0"
  env $E timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/products_shard0_$v.csv \
    python tools/shard_emulation.py --config products --shards 8 --only-shard 0 --reps 2 > /dev/null 2>&1
  env $E timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/reddit_fast_shard0_$v.csv \
    python tools/shard_emulation.py --config reddit --shards 8 --only-shard 0 --reps 2 --fast > /dev/null 2>&1
done
echo done > $OUT/done
