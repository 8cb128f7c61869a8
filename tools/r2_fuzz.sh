#!/bin/bash
set -u
OUT=gpurun_out/r2fuzz; mkdir -p $OUT
timeout 1200 python -m pytest tests/test_gpu_fuzz.py -q -x > $OUT/fuzz60.txt 2>&1
FUZZ_EXAMPLES=400 timeout 2400 python -m pytest tests/test_gpu_fuzz.py -q -x -k "device_plans or from_coo" > $OUT/fuzz400.txt 2>&1
echo done > $OUT/done
