#!/bin/bash
# exact-sum hub ring run alone (round-2 default): geometry sweep on Reddit 4/8 shards
set -u
OUT=gpurun_out/r2ring; mkdir -p $OUT
run() { tag=$1; shift; env "$@" timeout 600 python tools/shard_emulation.py --config reddit --shards 4,8 --reps 7 > $OUT/$tag.txt 2>&1; }
run default GESPMM_X=0
run small GESPMM_HUB_BIG=0
run small_c2 GESPMM_HUB_BIG=0 GESPMM_HUB_SPLIT=2
run c1 GESPMM_HUB_SPLIT=1
run c4 GESPMM_HUB_SPLIT=4
run vec2 GESPMM_HUB_VEC=2
run vec4 GESPMM_HUB_VEC=4
run vec4c4 GESPMM_HUB_VEC=4 GESPMM_HUB_SPLIT=4
echo done > $OUT/done
