#!/bin/bash
set -u
OUT=gpurun_out/r2flushclean; mkdir -p $OUT
for c in 0 1; do
  GESPMM_FLUSH_CLEAN=$c timeout 300 python bench.py --config pubmed --steps 20 --warmup 5 --no-cpu --no-e2e > $OUT/pubmed_$c.json 2> $OUT/pubmed_$c.log
  GESPMM_FLUSH_CLEAN=$c timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e --no-ceiling > $OUT/reddit_$c.json 2> $OUT/reddit_$c.log
done
echo done > $OUT/done
