#!/bin/bash
set -u
OUT=gpurun_out/e2eenv8; mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -q -x -k "pack or host or fuzz or io or dropin" > $OUT/pytest.txt 2>&1
run() { env "$@" timeout 300 python tools/e2e_env.py >> $OUT/env.txt 2>> $OUT/env.log; }
for rep in 1 2 3; do run GESPMM_X=0; done
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-ceiling > $OUT/bench.json 2> $OUT/bench.log
echo done > $OUT/done
