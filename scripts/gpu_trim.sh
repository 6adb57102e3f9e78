#!/bin/bash
# TMA maps stopping at K-1 / J-1 (HIMENO_TMA_TRIM): DRAM bytes of one L pass, then
# pass times on L / M / XL, one process per setting (maps are encoded at context creation)
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
for tr in 0 1 7; do
  echo "== ncu L HIMENO_TMA_TRIM=$tr"
  HIMENO_TMA_TRIM=$tr timeout 300 ncu --metrics $M --clock-control none -k regex:k_stencil_t -s 1 -c 1 --csv python scripts/ncu_tx_driver.py L 2>/dev/null | grep -E "gpu__time|dram__" | awk -F'","' '{print $(NF-2), $(NF-1), $NF}'
  echo "== ncu L single-step HIMENO_TMA_TRIM=$tr"
  HIMENO_TMA_TRIM=$tr HIMENO_SINGLE_STEP=1 timeout 300 ncu --metrics $M --clock-control none -k regex:k_stencil_tma -s 1 -c 1 --csv python scripts/ncu_tx_driver.py L 2>/dev/null | grep -E "gpu__time|dram__" | awk -F'","' '{print $(NF-2), $(NF-1), $NF}'
done
for r in 1 2; do
  for g in L M XL; do
    nn=40; [ $g = XL ] && nn=10
    for tr in 0 7; do
      HIMENO_TMA_TRIM=$tr GRID=$g NN=$nn python scripts/flow_exp.py "TRIM=$tr" 2>&1 | grep -v "^$" | tail -1
    done
  done
done
