#!/bin/bash
# round-2: low-degree rows-per-warp sweep (cold / warm graph / overlapped graph)
set -u
OUT=gpurun_out/r2rpw; mkdir -p $OUT
for n in 32 64 128 256; do for r in 1 2 4 8; do
  echo "n=$n rpw=$r $(timeout 300 python bench.py --config pubmed --n $n --rows-per-warp $r --steps 10 --warmup 3 --no-cpu --no-e2e --no-ceiling 2>>$OUT/log)" >> $OUT/sweep.txt
done; done
for r in 1 2 4 8; do
  echo "cora rpw=$r $(timeout 300 python bench.py --config cora --rows-per-warp $r --steps 10 --warmup 3 --no-cpu --no-e2e --no-ceiling 2>>$OUT/log)" >> $OUT/sweep.txt
done
echo done > $OUT/done
