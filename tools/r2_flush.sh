#!/bin/bash
set -u
OUT=gpurun_out/r2flush; mkdir -p $OUT
for rep in 1 2; do for mb in 512 256; do
  GESPMM_FLUSH_MB=$mb timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e > $OUT/f${mb}_$rep.json 2> $OUT/f${mb}_$rep.log
  sleep 5
done; done
echo done > $OUT/done
