#!/bin/bash
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_op_read.sum
for conf in "HIMENO_X=0" "HIMENO_TB2_FULL=0 HIMENO_TB2_CHUNK=32" "HIMENO_TB2_FULL=0 HIMENO_TB2_CHUNK=128" "HIMENO_TB2_FULL=0 HIMENO_TB2_CHUNK=16" "HIMENO_TB2_SHAPE=0" "HIMENO_TB2_SHAPE=2" "HIMENO_TB2_SHAPE=3" "HIMENO_TB2_STASH=0" "HIMENO_TMA_PROMO=2,2,0,0" "HIMENO_TMA_PROMO=2,2,1,1"; do
  echo "== $conf"
  env $conf timeout 300 ncu --metrics $M --clock-control none -k regex:k_stencil_tb2 -s 1 -c 1 --csv python scripts/ncu_tx_driver.py L 2>/dev/null | grep -E "gpu__time|dram__|lts__" | awk -F'","' '{print $(NF-2), $(NF-1), $NF}'
done
