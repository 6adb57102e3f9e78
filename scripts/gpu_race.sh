#!/bin/bash
TAG=${1:-race}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python scripts/sanitize_run.py > $OUT/racecheck.log 2>&1
grep -E "SUMMARY|Race reported" $OUT/racecheck.log | sort | uniq -c | head
timeout 300 python -m pytest tests -m gpu -q -x -k "temporal or stencil_config or headline" > $OUT/pytest.log 2>&1; tail -1 $OUT/pytest.log
bash scripts/gpu_tbchunk.sh 2>&1 | grep "chunk 64"
