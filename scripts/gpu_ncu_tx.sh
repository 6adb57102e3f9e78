#!/bin/bash
TAG=${1:-ncutx}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_stencil_tx -s 1 -c 1 \
  -o $OUT/tx python scripts/ncu_tx_driver.py L > $OUT/ncu.log 2>&1
tail -3 $OUT/ncu.log
HIMENO_TX=0 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_stencil_tb2 -s 1 -c 1 \
  -o $OUT/tb2 python scripts/ncu_tx_driver.py L > $OUT/ncu_tb2.log 2>&1
tail -3 $OUT/ncu_tb2.log
