set -u
OUT=gpurun_out/s6; mkdir -p $OUT
for v in "--config products" "--config products --l2-persist 2" "--config products --l2-persist 2 --l2-hot-mb 40" "--config products --l2-persist 2 --l2-hot-mb 100" "--config products --l2-hot-mb 40" "--config products --l2-hot-mb -1 --l2-persist 2" "--config products --hints 2" "--l2-persist 2" "--l2-persist 2 --l2-hot-mb 80"; do
  echo "== $v" >> $OUT/sweep.txt
  timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu $v 2>>$OUT/sweep.log | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['value'], d['roofline']['frac'], d['step_ms'], d['clocks']['sm_mhz'], d['config']['plan'])" >> $OUT/sweep.txt 2>&1
done
timeout 600 ncu --metrics lts__t_sector_hit_rate.pct,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum,lts__t_sectors_srcunit_tex_op_read.sum,gpu__time_duration.sum --clock-control none -k regex:k_warp -s 3 -c 1 --csv python bench.py --config products --steps 1 --warmup 3 --no-e2e --no-cpu > $OUT/ncu_default.csv 2>/dev/null
timeout 600 ncu --metrics lts__t_sector_hit_rate.pct,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum,lts__t_sectors_srcunit_tex_op_read.sum,gpu__time_duration.sum --clock-control none -k regex:k_warp -s 3 -c 1 --csv python bench.py --config products --steps 1 --warmup 3 --no-e2e --no-cpu --l2-persist 2 > $OUT/ncu_persist2.csv 2>/dev/null
