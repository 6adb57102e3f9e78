#!/bin/bash
TAG=${1:-r2}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -q -rf > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
tail -3 $OUT/pytest_gpu.log
for s in L XL M; do timeout 300 python scripts/sweep_stencil.py --size $s > $OUT/sweep_$s.jsonl 2>&1; done
grep -h '"cfg": [067]' $OUT/sweep_*.jsonl | cut -c1-110
timeout 900 python scripts/eval_all.py --size M --nn 3 --timeout 30 > $OUT/evalall_M.jsonl 2> $OUT/evalall_M.progress
tail -1 $OUT/evalall_M.jsonl | cut -c1-600
