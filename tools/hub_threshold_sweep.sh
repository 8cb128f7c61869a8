OUT=gpurun_out/r2_hubsweep3; mkdir -p $OUT
for t in 768 1024 1280 1536 1792; do
  timeout 300 python tools/shard_emulation.py --config reddit --shards 8 --reps 7 --hub-threshold $t > $OUT/t$t.txt 2>&1
done
