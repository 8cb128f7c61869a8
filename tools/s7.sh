set -u
OUT=gpurun_out/$1; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -3 > $OUT/pytest_parity.txt
shift
for v in "$@"; do
  echo "== $v" >> $OUT/sweep.txt
  timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu $v 2>>$OUT/sweep.log | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['value'], d['roofline']['frac'], d['step_ms'], d['clocks']['sm_mhz'], d['config']['plan'])" >> $OUT/sweep.txt 2>&1
done
