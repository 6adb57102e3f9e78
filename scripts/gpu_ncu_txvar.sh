#!/bin/bash
# DRAM bytes per exchange-kernel variant (one L two-step pass each)
OUT=gpurun_out/${1:-ncutxvar}
mkdir -p $OUT
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_op_write.sum,lts__t_sectors_op_read.sum
for conf in "HIMENO_TX=0" "HIMENO_TX=1" "HIMENO_TX_EVL=1" "HIMENO_TX_EVL=1 HIMENO_TX_DBG=1" "HIMENO_TX_DBG=3" "HIMENO_TX_EVL=1 HIMENO_TX_XRX=16 HIMENO_TX_AHEAD=1"; do
  echo "== $conf"
  env $conf timeout 300 ncu --metrics $M --clock-control none -k regex:k_stencil_t -s 1 -c 1 --csv python scripts/ncu_tx_driver.py L 2>/dev/null | grep -E "gpu__time|dram__|lts__"
done
