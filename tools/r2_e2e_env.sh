#!/bin/bash
set -u
OUT=gpurun_out/e2eenv10; mkdir -p $OUT
run() { env "$@" timeout 300 python tools/e2e_env.py >> $OUT/env.txt 2>> $OUT/env.log; }
for rep in 1 2 3; do
  run GESPMM_TAPER=1
  run GESPMM_TAPER=2
  run GESPMM_TAPER=2 GESPMM_CHUNKS=14
done
echo done > $OUT/done
