#!/bin/bash
set -u
OUT=gpurun_out/r2split2; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_split.py -q -x > $OUT/pytest.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -k "hub or fuzz or peer or parity" > $OUT/pytest_more.txt 2>&1
timeout 900 python tools/shard_emulation.py --config products --shards 1,4,8 --reps 5 > $OUT/products_split.txt 2>&1
GESPMM_HUB_SEGMENTS=0 timeout 900 python tools/shard_emulation.py --config products --shards 4,8 --reps 5 > $OUT/products_ring.txt 2>&1
timeout 900 python tools/shard_emulation.py --config reddit --shards 1,2,4,8 --reps 7 --fast > $OUT/reddit_fast_split.txt 2>&1
GESPMM_HUB_SEGMENTS=0 timeout 900 python tools/shard_emulation.py --config reddit --shards 2,4,8 --reps 7 --fast > $OUT/reddit_fast_ring.txt 2>&1
echo done > $OUT/done
