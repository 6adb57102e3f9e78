#!/bin/bash
# Two-step shape parity, GA throughput at host-core concurrency, config-5 transfer modes.
TAG=${1:-r3}
OUT=gpurun_out/$TAG
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
tail -2 $OUT/pytest_gpu.log
for w in 4 8 16; do
timeout 300 python -c "
import sys, json; sys.path.insert(0,'.')
import bench
print(json.dumps(bench.ga_throughput(0, 'M', 3, 20, 10, 0, $w)))
" >> $OUT/ga.jsonl 2>> $OUT/ga.err
done
cat $OUT/ga.jsonl
timeout 600 python scripts/transfer_modes.py --size M --nn 3 > $OUT/modes_M.jsonl 2> $OUT/modes_M.err
timeout 1200 python scripts/transfer_modes.py --size XL --nn 3 --repeats 2 > $OUT/modes_XL.jsonl 2> $OUT/modes_XL.err
tail -1 $OUT/modes_M.jsonl $OUT/modes_XL.jsonl; tail -3 $OUT/modes_XL.err
