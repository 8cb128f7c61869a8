#!/bin/bash
# Multi-rank paths on a single-GPU box: 2 ranks share cuda:0 over gloo.
OUT=gpurun_out/${1:-dist}; mkdir -p $OUT
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533"
timeout 600 python -m pytest tests/test_dist.py -m gpu -q -x 2>&1 | tail -3 > $OUT/pytest.txt
GESPMM_DIST_BACKEND=gloo timeout 600 $TR bench.py --gpus 2 --config pubmed --steps 5 --warmup 3 > $OUT/pubmed2.json 2> $OUT/pubmed2.log
GESPMM_DIST_BACKEND=gloo timeout 900 $TR bench.py --gpus 2 --steps 10 --warmup 3 > $OUT/reddit2.json 2> $OUT/reddit2.log
GESPMM_DIST_BACKEND=gloo timeout 900 $TR bench.py --gpus 2 --config gcn --steps 3 --warmup 3 > $OUT/gcn2.json 2> $OUT/gcn2.log
timeout 900 $TR bench.py --gpus 2 --impl reference --steps 2 --warmup 3 > $OUT/ref2.json 2> $OUT/ref2.log; echo "ref2 rc=$?" >> $OUT/pytest.txt
cat $OUT/pytest.txt; for f in pubmed2 reddit2 gcn2 ref2; do echo "== $f"; cut -c1-600 $OUT/$f.json; tail -2 $OUT/$f.log; done
