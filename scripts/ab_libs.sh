#!/bin/bash
# A/B of library builds (HIMENO_B200_LIB) on the device time loop: ROUNDS x libs x grids
# usage: bash scripts/ab_libs.sh "exp/lib_a.so exp/lib_b.so" "L M XL" [rounds]
LIBS=$1; GRIDS=${2:-"L M XL"}; ROUNDS=${3:-2}
for r in $(seq $ROUNDS); do
  for g in $GRIDS; do
    nn=40; [ $g = XL ] && nn=10
    for lib in $LIBS; do
      HIMENO_B200_LIB=$lib GRID=$g NN=$nn timeout 300 python scripts/flow_exp.py "LIB=$(basename $lib .so)" 2>&1 | grep -v "^$" | tail -1
    done
  done
done
