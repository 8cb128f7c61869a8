#!/bin/bash
# ncu --set full of one k_hub launch (148 hub rows x 21,657 nonzeros, N=128) per ring feed.
set -u
OUT=gpurun_out/${1:-r2_hub_ncu}; mkdir -p $OUT
python -c "import paper_2007_03179_b200" || exit 1
for feed in ldgsts g4; do
  GESPMM_HUB_FEED=$feed timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_hub -s 2 -c 1 \
    -o $OUT/hub_$feed -f python tools/longrow_probe.py --case 148,21657 --only hub --reps 1 > $OUT/ncu_$feed.log 2>&1
  python tools/ncu_summary.py $OUT/hub_$feed.ncu-rep $OUT/hub_$feed >> $OUT/ncu_$feed.log 2>&1
done
echo done > $OUT/done
