#!/bin/bash
# round-2 check: GPU suite + small-config lines
set -u
TAG=${1:-r2chk}
OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 2400 python -m pytest tests -m gpu -q -x -rs --durations=10 2>&1 | tail -60 > $OUT/pytest_gpu.txt
for a in "pubmed --n 128 --op sum" "pubmed --n 32 --op mean" "pubmed --n 64 --op max" "cora"; do
  timeout 300 python bench.py --config $a --steps 20 --warmup 5 --no-cpu --no-e2e >> $OUT/small.jsonl 2>> $OUT/small.log
done
echo done > $OUT/done
