#!/bin/bash
# ncu --set full of the split-hub-row launches on an 8-way products shard
# (segments k_warp, rest k_warp, combine) and of the overlap-chain small kernel
set -u
OUT=gpurun_out/r2splitfull; mkdir -p $OUT
timeout 1200 ncu --set full --clock-control none -k regex:"k_warp|k_split_combine" -s 3 -c 3 -o $OUT/prod_split -f \
  python tools/shard_emulation.py --config products --shards 8 --only-shard 0 --reps 1 > $OUT/ncu.log 2>&1
python tools/ncu_summary.py $OUT/prod_split.ncu-rep $OUT/prod_split > /dev/null 2>&1
find $OUT -name "*.ncu-rep" -size +30M -delete
echo done > $OUT/done
