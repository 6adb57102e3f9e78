#!/bin/bash
# BASELINE config 5 (transfer modes) at XL and M, plus the GA at host-core concurrency.
TAG=${1:-config5}
OUT=gpurun_out/$TAG
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python scripts/transfer_modes.py --size M --nn 3 > $OUT/modes_M.jsonl 2> $OUT/modes_M.err
timeout 1500 python scripts/transfer_modes.py --size XL --nn 3 > $OUT/modes_XL.jsonl 2> $OUT/modes_XL.err
tail -2 $OUT/modes_M.err $OUT/modes_XL.err
tail -1 $OUT/modes_M.jsonl $OUT/modes_XL.jsonl
