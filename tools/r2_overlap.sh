#!/bin/bash
# round-2: overlap_prev chains (parity) + small-config bench lines with the overlap replay
set -u
OUT=gpurun_out/r2ov2; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_overlap.py -q -x -rs > $OUT/pytest.txt 2>&1
for r in 1 2 4 8; do
  timeout 300 python bench.py --config pubmed --rows-per-warp $r --steps 20 --warmup 5 --no-cpu --no-e2e >> $OUT/rpw.jsonl 2>> $OUT/small.log
done
echo done > $OUT/done
