#!/bin/bash
# ncu --set full of the exact-sum hub ring run alone (8-way Reddit shard 0)
set -u
OUT=gpurun_out/r2hubncu; mkdir -p $OUT
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_hub -s 1 -c 1 -o $OUT/hub -f \
  python tools/shard_emulation.py --config reddit --shards 8 --only-shard 0 --reps 2 > $OUT/ncu.log 2>&1
python tools/ncu_summary.py $OUT/hub.ncu-rep $OUT/hub_summary > /dev/null 2>&1
ncu -i $OUT/hub.ncu-rep --page details --csv > $OUT/hub_details.csv 2>/dev/null
find $OUT -name "*.ncu-rep" -size +30M -delete
echo done > $OUT/done
