#!/bin/bash
# round-2 session b: hub feed ncu (both feeds), products L2 hit-rate study (default,
# hot map 80 MB, hints off), headline launch list + ncu full of this round's kernel.
set -u
OUT=gpurun_out/r2b; mkdir -p $OUT
python -c "import paper_2007_03179_b200" || exit 1
for feed in ldgsts g4; do
  GESPMM_HUB_FEED=$feed timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_hub -s 2 -c 1 \
    -o $OUT/hub_$feed -f python tools/longrow_probe.py --case 148,21657 --only hub --reps 4 > $OUT/ncu_hub_$feed.log 2>&1
  python tools/ncu_summary.py $OUT/hub_$feed.ncu-rep $OUT/hub_$feed >> $OUT/ncu_hub_$feed.log 2>&1
done
for v in "def:" "hot80:--l2-hot-mb 80" "nohints:--no-hints"; do
  tag=${v%%:*}; extra=${v#*:}
  GESPMM_EXPERIMENTAL=1 timeout 900 ncu --section SpeedOfLight --section MemoryWorkloadAnalysis --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum,lts__t_sectors_srcunit_tex_op_read.sum \
    --clock-control none -k regex:k_warp -s 3 -c 1 -o $OUT/prod_$tag -f \
    python bench.py --config products --steps 1 --warmup 3 --no-e2e --no-cpu $extra > /dev/null 2> $OUT/prod_$tag.log
  python tools/ncu_summary.py $OUT/prod_$tag.ncu-rep $OUT/prod_$tag >> $OUT/prod_$tag.log 2>&1
  GESPMM_EXPERIMENTAL=1 timeout 300 python bench.py --config products --steps 10 --warmup 3 --no-e2e --no-cpu $extra > $OUT/prod_bench_$tag.json 2>> $OUT/prod_$tag.log
done
bash tools/ncu_capture.sh r2_reddit
mv gpurun_out/ncu_r2_reddit $OUT/
python tools/ncu_summary.py $OUT/ncu_r2_reddit/prof.ncu-rep $OUT/reddit_full > /dev/null 2>&1
# keep the merge under gpurun's 64 MiB: summaries stay, big reports go
find $OUT -name "*.ncu-rep" -size +20M -delete
find $OUT -name "prod_*.ncu-rep" -delete
du -sh $OUT > $OUT/du.txt
echo done > $OUT/done
