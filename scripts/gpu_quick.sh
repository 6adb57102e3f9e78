#!/bin/bash
# Quick GPU iteration: gpu tests + stencil sweep (+ optional extra command).
TAG=${1:-quick}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
for s in L M XL; do timeout 300 python scripts/sweep_stencil.py --size $s > $OUT/sweep_$s.jsonl 2>&1; done
tail -3 $OUT/pytest_gpu.log
cat $OUT/sweep_*.jsonl
