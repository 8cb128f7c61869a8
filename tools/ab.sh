#!/bin/bash
# A/B bench sweep: bash tools/ab.sh <tag> "<LIBVARIANT>|<bench args>" ...
# LIBVARIANT: "" = in-tree lib, else build/variants/<name>/libgespmm.so
set -u
OUT=gpurun_out/$1; shift; mkdir -p $OUT
for spec in "$@"; do
  var=${spec%%|*}; args=${spec#*|}
  lib=""; [ -n "$var" ] && lib=$PWD/build/variants/$var/libgespmm.so
  echo "== [$var] $args" >> $OUT/sweep.txt
  GESPMM_LIB=$lib timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu $args 2>>$OUT/sweep.log | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['value'], d['roofline']['frac'], d['step_ms'], d['clocks']['sm_mhz'], d['config']['plan'][:60])" >> $OUT/sweep.txt 2>&1
done
