#!/bin/bash
set -u
OUT=gpurun_out/r2hubseq3; mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -q -x -k "hub or fuzz or shard or host or split" > $OUT/pytest.txt 2>&1
timeout 600 python tools/shard_emulation.py --config reddit --shards 1,2,4,8 --reps 7 > $OUT/reddit.txt 2>&1
GESPMM_HUB_SEQ=0 GESPMM_HUB_PERSIST=2 timeout 600 python tools/shard_emulation.py --config reddit --shards 4,8 --reps 7 > $OUT/reddit_old.txt 2>&1
for i in 1 2; do timeout 300 python tools/e2e_env.py >> $OUT/e2e.txt 2>>$OUT/e2e.log; GESPMM_HUB_SEQ=0 GESPMM_HUB_PERSIST=2 timeout 300 python tools/e2e_env.py >> $OUT/e2e.txt 2>>$OUT/e2e.log; done
echo done > $OUT/done
