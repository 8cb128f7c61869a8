#!/bin/bash
# round-2: e2e with the vectorised packer (+ packed-upload parity tests)
set -u
TAG=${1:-r2e2e}
OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -q -x -k "pack or host or fuzz" > $OUT/pytest.txt 2>&1
for i in 1 2; do
  timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-ceiling > $OUT/bench$i.json 2> $OUT/bench$i.log
done
for t in 8 12 16; do
  GESPMM_PACK_THREADS=$t timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-ceiling > $OUT/bench_t$t.json 2> $OUT/bench_t$t.log
done
echo done > $OUT/done
