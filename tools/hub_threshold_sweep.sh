OUT=gpurun_out/r2_hubsweep; mkdir -p $OUT
for t in 0 2048 2600 3200 4096 5000 7000; do
  timeout 300 python tools/shard_emulation.py --config reddit --shards 8 --reps 7 --hub-threshold $t > $OUT/t$t.txt 2>&1
done
