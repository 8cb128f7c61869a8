#!/bin/bash
# Relocated hot rows: parity at products scale + budget / policy sweep (products).
set -u
OUT=gpurun_out/${1:-r2_reloc}; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_fullscale.py -m gpu -q -x -k "products" 2>&1 | tail -5 > $OUT/pytest_products.txt
run() { # tag, env, args
  env GESPMM_EXPERIMENTAL=1 $2 timeout 300 python bench.py --config products --steps 10 --warmup 3 --no-e2e --no-cpu $3 > $OUT/prod_$1.json 2> $OUT/prod_$1.log
  echo "products $1: $(grep per-step $OUT/prod_$1.log | tail -1)" >> $OUT/summary.txt
}
run off "X=1" "--hot-rows-mb -1"
for mode in 1 2 0; do for mb in 40 80 110; do run m${mode}_$mb "GESPMM_RELOC_POLICY=$mode" "--hot-rows-mb $mb"; done; done
run off2 "X=1" "--hot-rows-mb -1"
echo done > $OUT/done
