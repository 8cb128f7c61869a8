#!/bin/bash
# Hub ring feed A/B: TMA gather4 (default) vs LDGSTS producer warps.
#   bash tools/hub_ab.sh <tag> [tests]
set -u
TAG=$1; shift
OUT=gpurun_out/$TAG; mkdir -p $OUT
if [ "${1:-}" = "tests" ]; then
  timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -m gpu -q -x -k "hub or fuzz" 2>&1 | tail -15 > $OUT/pytest_hub.txt
fi
for feed in g4 ldgsts g4 ldgsts; do
  GESPMM_HUB_FEED=$feed timeout 300 python tools/shard_emulation.py --config reddit --shards 8 --reps 9 >> $OUT/shard8_$feed.txt 2>&1
done
for feed in g4 ldgsts; do
  GESPMM_HUB_FEED=$feed timeout 300 python tools/longrow_probe.py --only hub > $OUT/longrow_$feed.txt 2>&1
  GESPMM_HUB_FEED=$feed timeout 300 python tools/shard_emulation.py --config reddit --shards 2,4 --reps 7 > $OUT/shard24_$feed.txt 2>&1
done
echo done > $OUT/done
