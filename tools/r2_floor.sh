#!/bin/bash
set -u
OUT=gpurun_out/r2seqall; mkdir -p $OUT
timeout 600 python tools/shard_emulation.py --config reddit --shards 1,2,4,8 --reps 7 > $OUT/reddit.txt 2>&1
timeout 900 python tools/shard_emulation.py --config products --shards 2,4,8 --reps 5 > $OUT/products.txt 2>&1
for i in 1 2; do timeout 300 python tools/e2e_env.py >> $OUT/e2e.txt 2>>$OUT/e2e.log; done
timeout 600 python bench.py --config gcn --steps 10 --warmup 3 > $OUT/gcn.json 2> $OUT/gcn.log
timeout 900 python -m pytest tests -m gpu -q -x -k "hub or shard or split or fuzz or peer or dist" > $OUT/pytest.txt 2>&1
echo done > $OUT/done
