#!/bin/bash
# Host-loop timing (all-CPU and mixed genomes) + GA throughput, after host-loop changes.
TAG=${1:-host}
OUT=gpurun_out/$TAG
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
tail -2 $OUT/pytest_gpu.log
timeout 300 python -c "
import sys; sys.path.insert(0,'.')
from paper_2002_12115_b200.evaluator import B200Evaluator
with B200Evaluator('M', nn=3) as ev:
    for g in ('0000000000000','1001000000000','0000000000001','0000000100000','1001001000000'):
        g=tuple(int(c) for c in g)
        ts=[ev.measure(g).seconds for _ in range(3)]
        st=ev.stats[g]
        print(''.join(map(str,g)), ['%.4f'%t for t in ts], 'host_s %.4f'%st['host_s'])
" 2>&1 | tee $OUT/host_times.txt
for w in 4 16; do
timeout 300 python -c "
import sys, json; sys.path.insert(0,'.')
import bench
print(json.dumps(bench.ga_throughput(0, 'M', 3, 20, 10, 0, $w)))
" >> $OUT/ga.jsonl 2>> $OUT/ga.err
done
cat $OUT/ga.jsonl
