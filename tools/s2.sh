set -u
OUT=gpurun_out/s2; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "column_slices or tuned_shapes or hub_rows" 2>&1 | tail -5 > $OUT/pytest_slices.txt
timeout 600 python -m pytest tests/test_gpu_sectors.py -q -x 2>&1 | grep -v "^| .*yes.*yes" | tail -60 > $OUT/pytest_sectors.txt
export SWEEP_LIST
for v in "--config products --col-slices 1" "--config products --col-slices 2" "--config products --col-slices 4" "--config products --col-slices 8" "--config products --col-slices 8 --l2-hot-mb -1" "--config products --col-slices 4 --l2-hot-mb -1" "--col-slices 1" "--col-slices 2" "--col-slices 4"; do
  echo "== $v" >> $OUT/sweep.txt
  timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu $v 2>>$OUT/sweep.log | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['value'], d['roofline']['frac'], d['step_ms'], d['clocks']['sm_mhz'], d['config']['plan'])" >> $OUT/sweep.txt 2>&1
done
