#!/bin/bash
set -u
OUT=gpurun_out/r2coo; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_coo.py -q -x -rs > $OUT/pytest.txt 2>&1
timeout 900 python tools/coo_time.py --products > $OUT/coo_time.jsonl 2> $OUT/coo_time.log
echo done > $OUT/done
