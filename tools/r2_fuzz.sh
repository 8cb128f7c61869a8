#!/bin/bash
set -u
OUT=gpurun_out/r2fuzz2; mkdir -p $OUT
FUZZ_EXAMPLES=1500 timeout 3000 python -m pytest tests/test_gpu_fuzz.py -q -x -p no:cacheprovider > $OUT/fuzz1500.txt 2>&1
echo done > $OUT/done
