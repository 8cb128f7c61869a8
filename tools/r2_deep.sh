#!/bin/bash
# round-2: deeper gather batch (U=16) for full-warp CF=1 rows: whole matrix and 8 shards
set -u
OUT=gpurun_out/r2deep; mkdir -p $OUT
for v in default uw16 uw16b5; do
  if [ $v = default ]; then L=""; else L="GESPMM_LIB=build/variants/$v/libgespmm.so"; fi
  env $L timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-ceiling > $OUT/bench_$v.json 2>$OUT/bench_$v.log
  for t in 2048 4096 6000 8000; do
    env $L timeout 300 python tools/shard_emulation.py --config reddit --shards 8 --reps 7 --hub-threshold $t > $OUT/shard8_${v}_t$t.txt 2>&1
  done
  env $L timeout 300 python tools/shard_emulation.py --config reddit --shards 2,4 --reps 7 > $OUT/shard24_${v}.txt 2>&1
done
echo done > $OUT/done
