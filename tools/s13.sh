OUT=gpurun_out/s13; mkdir -p $OUT
for cfg in "1 4" "2 4" "2 8"; do set -- $cfg
timeout 600 ncu --set full --clock-control none -k regex:"k_warp|k_stream" -s 3 -c 1 -o $OUT/pubmed_rs$1_rpw$2 -f python bench.py --config pubmed --steps 1 --warmup 3 --no-e2e --no-cpu --row-stream $1 --rows-per-warp $2 > /dev/null 2> $OUT/ncu_$1_$2.log
done
bash tools/ab.sh s13 "|--config pubmed --no-flush --rows-per-warp 1 --row-stream 1" "|--config pubmed --no-flush --rows-per-warp 4 --row-stream 1" "|--config pubmed --no-flush --rows-per-warp 8 --row-stream 2"
