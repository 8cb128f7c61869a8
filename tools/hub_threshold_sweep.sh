OUT=gpurun_out/r2_hubsweep4; mkdir -p $OUT
for t in 3000 4000 5000 6000 8000; do
  timeout 300 python tools/shard_emulation.py --config reddit --shards 2 --reps 7 --hub-threshold $t > $OUT/t$t.txt 2>&1
done
for t in 3500 4096 5000; do
  timeout 300 python tools/shard_emulation.py --config reddit --shards 4 --reps 7 --hub-threshold $t > $OUT/q$t.txt 2>&1
done
