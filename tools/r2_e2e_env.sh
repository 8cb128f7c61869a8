#!/bin/bash
set -u
OUT=gpurun_out/e2eenv9; mkdir -p $OUT
timeout 600 python -m pytest tests -m gpu -q -x -k "pack" > $OUT/pytest.txt 2>&1
GESPMM_PACK_RING=3 timeout 600 python -m pytest tests -m gpu -q -x -k "pack or host" >> $OUT/pytest.txt 2>&1
run() { env "$@" timeout 300 python tools/e2e_env.py >> $OUT/env.txt 2>> $OUT/env.log; }
for rep in 1 2; do
  run GESPMM_X=0
  run GESPMM_PACK_RING=2
  run GESPMM_PACK_RING=3
  run GESPMM_PACK_RING=4
done
echo done > $OUT/done
