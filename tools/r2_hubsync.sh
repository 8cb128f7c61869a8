#!/bin/bash
set -u
OUT=gpurun_out/r2hubsync; mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -q -x -k "hub or fuzz or shard" > $OUT/pytest.txt 2>&1
for rep in 1; do for v in default; do
  if [ $v = default ]; then L=""; else L="GESPMM_LIB=build/variants/$v/libgespmm.so"; fi
  env $L timeout 300 python tools/shard_emulation.py --config reddit --shards 2,4,8 --reps 7 > $OUT/shard_${v}_$rep.txt 2>&1
  env $L timeout 300 python tools/longrow_probe.py --case 148,21657 --only hub --reps 4 > $OUT/longrow_${v}_$rep.txt 2>&1
done; done
timeout 1500 compute-sanitizer --tool racecheck --target-processes all --print-limit 20 python tools/sanitize_driver.py > $OUT/racecheck.txt 2>&1
echo done > $OUT/done
