#!/bin/bash
set -u
OUT=gpurun_out/r2n44; mkdir -p $OUT
for n in 44 256; do
  timeout 300 python bench.py --n $n --steps 10 --warmup 3 --no-cpu --no-e2e --no-ceiling > $OUT/seq_$n.json 2> $OUT/seq_$n.log
  GESPMM_HUB_SEQ=0 GESPMM_HUB_PERSIST=2 timeout 300 python bench.py --n $n --steps 10 --warmup 3 --no-cpu --no-e2e --no-ceiling > $OUT/old_$n.json 2> $OUT/old_$n.log
done
GESPMM_HUB_SEQ=0 GESPMM_HUB_PERSIST=2 timeout 600 python bench.py --config gcn --steps 10 --warmup 3 > $OUT/gcn_old.json 2> $OUT/gcn_old.log
timeout 600 python bench.py --config gcn --steps 10 --warmup 3 > $OUT/gcn_seq.json 2> $OUT/gcn_seq.log
echo done > $OUT/done
