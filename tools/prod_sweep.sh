#!/bin/bash
# products (N=256 max+arg) shape sweep + GCN step + ncu DRAM bytes with the hot map.
OUT=gpurun_out/${1:-prod}; mkdir -p $OUT
run() { local name=$1; shift
  timeout 400 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu "$@" > $OUT/$name.json 2> $OUT/$name.log
  python -c "import json;d=json.load(open('$OUT/$name.json'));print('$name', d['ms_per_step'], d['step_ms'], d['clocks']['sm_mhz'], d['config'].get('plan'))" >> $OUT/summary.txt 2>&1 || echo "$name FAILED" >> $OUT/summary.txt
}
for cf in 1 2 4; do
  run p_cf${cf}_hot --config products --tuned-cf $cf
  run p_cf${cf}_off --config products --tuned-cf $cf --l2-hot-mb -1
done
true
timeout 600 python bench.py --config gcn --steps 5 --warmup 3 > $OUT/gcn.json 2> $OUT/gcn.log; cat $OUT/gcn.json >> $OUT/summary.txt
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex_op_read.sum --clock-control none -k regex:k_warp -c 2 --csv \
  python bench.py --config products --steps 1 --warmup 1 --no-e2e --no-cpu > $OUT/ncu_hot.csv 2> $OUT/ncu_hot.log
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex_op_read.sum --clock-control none -k regex:k_warp -c 2 --csv \
  python bench.py --config products --steps 1 --warmup 1 --no-e2e --no-cpu --l2-hot-mb -1 > $OUT/ncu_off.csv 2> $OUT/ncu_off.log
cat $OUT/summary.txt
