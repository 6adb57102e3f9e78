#!/bin/bash
OUT=gpurun_out/${1:-ncutxdbg}
mkdir -p $OUT
for d in 1 3 0; do
  HIMENO_TX=1 HIMENO_TX_DBG=$d timeout 600 ncu --set full --clock-control none --import-source on \
    -k regex:k_stencil_tx -s 1 -c 1 -o $OUT/tx_dbg$d python scripts/ncu_tx_driver.py L > $OUT/ncu_dbg$d.log 2>&1
  tail -1 $OUT/ncu_dbg$d.log
done
