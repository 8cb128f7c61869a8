#!/bin/bash
# One GPU session: parity tests, ceilings, bench sweeps, ncu launch list + full captures.
# Usage (on the box via gpurun): bash tools/gpu_session.sh <tag> [sections...]
set -u
TAG=${1:-s}; shift || true
SECTIONS=${@:-"tests ceilings sweep ncu"}
OUT=gpurun_out/$TAG; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/gpu.txt 2>&1
for s in $SECTIONS; do case $s in
tests)
  timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > $OUT/pytest_gpu.txt
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.txt 2>&1 ;;
fasttests)
  timeout 900 python -m pytest tests -m gpu -q -x -k "not slow" 2>&1 | tail -15 > $OUT/pytest_gpu.txt ;;
ceilings)
  timeout 600 python tools/ceilings.py --json $OUT/ceilings.json > $OUT/ceilings.txt 2>&1 ;;
sweep)
  for v in ${SWEEP:-"--variant tuned" "--variant tuned --fast" "--variant tuned --hub-threshold 7884" \
           "--variant crc-cwm --cf 2" "--variant crc-cwm --cf 4" "--variant crc-cwm --cf 8" "--variant crc" "--variant naive" \
           "--config products" "--config pubmed"}; do
    echo "== $v" >> $OUT/sweep.txt
    timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu $v 2>>$OUT/sweep.log | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['value'], d['roofline']['frac'], d['config']['plan'])" >> $OUT/sweep.txt 2>&1
  done ;;
bench)
  timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.log ;;
ncu)
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
      python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu > $OUT/ncu_launch_bench.json 2> $OUT/ncu_launch.log
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_warp -s 2 -c 1 -o $OUT/prof_warp -f \
      python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > /dev/null 2> $OUT/ncu_warp.log
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_cta -s 2 -c 1 -o $OUT/prof_cta -f \
      python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > /dev/null 2> $OUT/ncu_cta.log ;;
esac; done
echo "session $TAG done"
