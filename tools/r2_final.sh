#!/bin/bash
# round-2 closing measurements at HEAD: GPU suite, smoke, bench (ours + reference),
# shard emulation (Reddit, products), launch list + ncu --set full of k_warp
set -u
OUT=gpurun_out/${TAG:-r2e}; mkdir -p $OUT
bash tools/gpu_r2.sh ${TAG:-r2e} tests smoke bench
timeout 600 python tools/shard_emulation.py --config reddit --shards 1,2,4,8 --reps 7 > $OUT/shard_reddit.txt 2>&1
timeout 900 python tools/shard_emulation.py --config products --shards 1,2,4,8 --reps 5 > $OUT/shard_products.txt 2>&1
bash tools/ncu_capture.sh ${TAG:-r2e}_reddit
python tools/ncu_summary.py gpurun_out/ncu_${TAG:-r2e}_reddit/prof.ncu-rep $OUT/ncu_full_k_warp_reddit > /dev/null 2>&1
find gpurun_out/ncu_${TAG:-r2e}_reddit -name "*.ncu-rep" -size +30M -delete
echo done > $OUT/done
