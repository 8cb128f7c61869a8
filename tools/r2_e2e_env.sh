#!/bin/bash
set -u
OUT=gpurun_out/e2eenv4; mkdir -p $OUT
run() { env "$@" timeout 300 python tools/e2e_env.py >> $OUT/env.txt 2>> $OUT/env.log; }
for rep in 1 2 3; do
  run GESPMM_X=0
  run GESPMM_HOST_POLL=0
  run GESPMM_HOST_POLL=1
  run GESPMM_HOST_POLL=4
done
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-ceiling > $OUT/bench.json 2> $OUT/bench.log
echo done > $OUT/done
