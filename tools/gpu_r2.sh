#!/bin/bash
# Round-2 GPU session: full -m gpu suite (incl. full-scale parity, 2-rank bench), smoke, bench.
set -u
TAG=${1:-r2}; shift || true
SECTIONS=${@:-"tests smoke bench"}
OUT=gpurun_out/$TAG; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/gpu.txt 2>&1
nproc >> $OUT/gpu.txt; grep -m1 "model name" /proc/cpuinfo >> $OUT/gpu.txt
for s in $SECTIONS; do case $s in
tests)
  timeout 2400 python -m pytest tests -m gpu -q -x --durations=15 2>&1 | tail -40 > $OUT/pytest_gpu.txt ;;
fast)
  timeout 1500 python -m pytest tests -m "gpu and not slow" -q -x 2>&1 | tail -30 > $OUT/pytest_gpu.txt ;;
full)
  timeout 1500 python -m pytest tests/test_gpu_fullscale.py tests/test_gpu_bench_contract.py -q -x --durations=10 2>&1 | tail -30 > $OUT/pytest_full.txt ;;
smoke)
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.txt 2>&1 ;;
bench)
  timeout 900 python bench.py --steps 20 --warmup 5 > $OUT/bench.json 2> $OUT/bench.log
  timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > $OUT/ref.json 2> $OUT/ref.log ;;
esac; done
echo "session $TAG done"
