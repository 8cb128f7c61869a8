#!/bin/bash
# Step-time drift probe: same bench with/without the nvidia-smi sampler and at
# two sampling intervals; per-step ms go to stderr logs under gpurun_out/$1.
OUT=gpurun_out/${1:-clk}; mkdir -p $OUT
B="python bench.py --steps 100 --warmup 5 --no-e2e --no-cpu"
GESPMM_NO_CLOCKS=1 timeout 300 $B > $OUT/noclk.json 2> $OUT/noclk.log
GESPMM_CLOCK_MS=20 timeout 300 $B > $OUT/clk20.json 2> $OUT/clk20.log
GESPMM_CLOCK_MS=200 timeout 300 $B > $OUT/clk200.json 2> $OUT/clk200.log
GESPMM_NO_CLOCKS=1 timeout 300 $B --no-flush > $OUT/noflush.json 2> $OUT/noflush.log
nvidia-smi -q -d CLOCK,PERFORMANCE,TEMPERATURE,POWER > $OUT/smi.txt 2>&1
for f in noclk clk20 clk200 noflush; do echo "== $f"; grep "per-step" $OUT/$f.log | cut -c1-2000; python -c "import json;d=json.load(open('$OUT/$f.json'));print(d['ms_per_step'],d['step_ms'],d['clocks'])"; done
