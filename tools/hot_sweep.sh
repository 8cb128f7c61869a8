#!/bin/bash
# Hot-column L2 map sweep: products (max+arg, N=256) and Reddit (sum, N=128).
OUT=gpurun_out/${1:-hot}; mkdir -p $OUT
run() { # name, args...
  local name=$1; shift
  GESPMM_NO_CLOCKS=1 timeout 400 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu "$@" \
     > $OUT/$name.json 2> $OUT/$name.log
  python -c "import json;d=json.load(open('$OUT/$name.json'));print('$name', d['ms_per_step'], d['step_ms'], d['config']['plan'])" >> $OUT/summary.txt 2>&1 || echo "$name FAILED" >> $OUT/summary.txt
}
for cfg in ${CFGS:-products reddit}; do
  run ${cfg}_off --config $cfg --l2-hot-mb -1
  run ${cfg}_auto --config $cfg
  for mb in ${MBS:-40 100}; do run ${cfg}_mb$mb --config $cfg --l2-hot-mb $mb; done
  run ${cfg}_auto_h2 --config $cfg --hints 2
done
cat $OUT/summary.txt
# drift diagnostics: clock log at 20 ms and no-hints run
GESPMM_CLOCK_MS=20 GESPMM_CLOCK_LOG=$OUT/clocklog.csv timeout 300 python bench.py --steps 100 --warmup 3 --no-e2e --no-cpu > $OUT/drift.json 2> $OUT/drift.log
GESPMM_NO_CLOCKS=1 timeout 300 python bench.py --steps 100 --warmup 3 --no-e2e --no-cpu --no-hints > $OUT/drift_nohints.json 2> $OUT/drift_nohints.log
grep per-step $OUT/drift.log $OUT/drift_nohints.log | cut -c1-900
