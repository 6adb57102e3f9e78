#!/bin/bash
TAG=${1:-ncu_tb2}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_stencil_tb2 -s 2 -c 1 \
  -o $OUT/tb2 python scripts/sweep_stencil.py --size L --reps 1 > $OUT/ncu.log 2>&1
tail -3 $OUT/ncu.log
