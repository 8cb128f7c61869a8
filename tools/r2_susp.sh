#!/bin/bash
set -u
OUT=gpurun_out/r2susp; mkdir -p $OUT
for v in default susp200 susp1000 susp5000; do
  if [ $v = default ]; then L=""; else L="GESPMM_LIB=build/variants/$v/libgespmm.so"; fi
  env $L timeout 600 python tools/shard_emulation.py --config reddit --shards 2,4,8 --reps 7 > $OUT/$v.txt 2>&1
  env $L timeout 300 python tools/longrow_probe.py --case 148,21657 --only hub --reps 4 > $OUT/longrow_$v.txt 2>&1
done
echo done > $OUT/done
