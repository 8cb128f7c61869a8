#!/bin/bash
# round-2: propagate config (fused vs NCCL-style exchange) test + Reddit lines
set -u
OUT=gpurun_out/r2prop; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_bench_contract.py -q -x -k propagate > $OUT/pytest.txt 2>&1
for ex in fused nccl; do
  timeout 600 python bench.py --config propagate --exchange $ex --steps 5 --warmup 3 > $OUT/reddit_1_$ex.json 2> $OUT/reddit_1_$ex.log
  GESPMM_DIST_BACKEND=gloo timeout 900 python bench.py --gpus 2 --config propagate --exchange $ex --steps 5 --warmup 3 > $OUT/reddit_2_$ex.json 2> $OUT/reddit_2_$ex.log
done
echo done > $OUT/done
