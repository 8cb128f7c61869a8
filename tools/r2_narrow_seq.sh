#!/bin/bash
set -u
OUT=gpurun_out/r2narrowseq; mkdir -p $OUT
for n in 32 44 64 96; do
  timeout 300 python bench.py --n $n --steps 10 --warmup 3 --no-cpu --no-e2e --no-ceiling > $OUT/on_$n.json 2> $OUT/on_$n.log
  GESPMM_HUB_SEQ_ALWAYS=0 timeout 300 python bench.py --n $n --steps 10 --warmup 3 --no-cpu --no-e2e --no-ceiling > $OUT/off_$n.json 2> $OUT/off_$n.log
done
echo done > $OUT/done
