OUT=gpurun_out/r2_reloc_ncu; mkdir -p $OUT
for mb in -1 80; do
timeout 900 ncu --section SpeedOfLight --section MemoryWorkloadAnalysis --section WarpStateStats --section SchedulerStats --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum,lts__average_gcomp_input_sector_success_rate.pct \
    --clock-control none -k regex:k_warp -s 3 -c 1 -o $OUT/prod_$mb -f \
    python bench.py --config products --steps 1 --warmup 3 --no-e2e --no-cpu --hot-rows-mb $mb > /dev/null 2> $OUT/prod_$mb.log
python tools/ncu_summary.py $OUT/prod_$mb.ncu-rep $OUT/prod_$mb >> $OUT/prod_$mb.log 2>&1
ncu -i $OUT/prod_$mb.ncu-rep --page details --csv > $OUT/prod_${mb}_details.csv 2>/dev/null
rm -f $OUT/prod_$mb.ncu-rep
done
