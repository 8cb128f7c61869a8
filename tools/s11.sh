OUT=gpurun_out/s11; mkdir -p $OUT
for rs in 1 2; do
timeout 600 ncu --set full --clock-control none -k regex:"k_warp|k_stream" -s 3 -c 1 -o $OUT/pubmed_rs$rs -f python bench.py --config pubmed --steps 1 --warmup 3 --no-e2e --no-cpu --row-stream $rs > /dev/null 2> $OUT/ncu_$rs.log
done
timeout 300 nsys --version > $OUT/nsys.txt 2>&1
