#!/bin/bash
# One ncu --set full capture of the first timed k_warp launch of a bench config
# (1 GPU), plus the launch list of the same command.
#   bash tools/ncu_capture.sh <tag> <bench args...>
set -u
TAG=$1; shift
OUT=gpurun_out/ncu_$TAG; mkdir -p $OUT
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
    python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu "$@" > $OUT/launch_bench.json 2> $OUT/launch.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_warp -s 3 -c 1 -o $OUT/prof -f \
    python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu "$@" > /dev/null 2> $OUT/ncu.log
echo done > $OUT/done
