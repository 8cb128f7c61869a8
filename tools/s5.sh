set -u
OUT=gpurun_out/s5; mkdir -p $OUT
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu > $OUT/ncu_launch_bench.json 2> $OUT/ncu_launch.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_warp -s 2 -c 1 -o $OUT/prof_products -f python bench.py --config products --steps 2 --warmup 3 --no-e2e --no-cpu > /dev/null 2> $OUT/ncu_products.log
timeout 1800 python -m pytest tests -m "gpu and slow" -q -x 2>&1 | tail -5 > $OUT/pytest_slow.txt
timeout 600 python build/../bench.py --impl reference --steps 5 --warmup 3 > $OUT/bench_ref.json 2> $OUT/bench_ref.log
echo done
