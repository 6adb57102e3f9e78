#!/bin/bash
# exchange-kernel check: its parity tests, L/M parity, A/B timing, ncu launch list
TAG=${1:-tx}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "exchange or headline or m_grid or temporal" > $OUT/pytest_tx.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_tx.log
tail -3 $OUT/pytest_tx.log
timeout 300 python scripts/tx_ab.py M,L,XL 3 > $OUT/ab.txt 2>&1; cat $OUT/ab.txt
