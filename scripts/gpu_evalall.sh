#!/bin/bash
TAG=${1:-evalall}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 1200 python scripts/eval_all.py --size M --nn 3 --timeout 30 > $OUT/evalall_M.jsonl 2> $OUT/evalall_M.progress
tail -3 $OUT/evalall_M.jsonl
