#!/bin/bash
TAG=${1:-sanitize}
OUT=gpurun_out/$TAG
mkdir -p $OUT
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_run.py > $OUT/$tool.log 2>&1
  echo "$tool rc=$?" >> $OUT/$tool.log
  echo "== $tool"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|rc=|Error" $OUT/$tool.log | head -5
done
# the tile-exchange kernel alone (its CTAs wait on each other; instrumented code must
# still fit one CTA per SM)
for tool in memcheck racecheck synccheck; do
  SANITIZE_TX=1 timeout 900 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_run.py > $OUT/tx_$tool.log 2>&1
  echo "tx $tool rc=$?" >> $OUT/tx_$tool.log
  echo "== tx $tool"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|rc=|Error|^tx " $OUT/tx_$tool.log | head -5
done
