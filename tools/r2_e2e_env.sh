#!/bin/bash
set -u
OUT=gpurun_out/e2eenv2; mkdir -p $OUT
run() { env "$@" timeout 300 python tools/e2e_env.py >> $OUT/env.txt 2>> $OUT/env.log; }
for rep in 1 2; do
  for c in 12 16 20 24 8; do run GESPMM_CHUNKS=$c; done
done
echo done > $OUT/done
