#!/bin/bash
# Round-2 evidence: launch list of the bench command, ncu --set full of the headline
# two-step pass (L) and of the M flow launch, and the tx kernel on L.
TAG=${1:-prof2}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $OUT/launches.csv python bench.py --steps 2 --warmup 3 --no-ga --no-cpu-baseline \
  --no-other-grids --no-ft > $OUT/bench_under_ncu.log 2>&1
echo "launch list rc=$?"
cat > /tmp/mflow.py <<'PY'
import sys; sys.path.insert(0,'.')
from paper_2002_12115_b200 import native as N
from paper_2002_12115_b200.apps import himeno
sz = himeno.size(sys.argv[1])
with N.Context(0, sz.I, sz.J, sz.K) as c:
    c.init_device(); c.jacobi_device(int(sys.argv[2]), 1)
    print(N.last_two_step_kernel(), c.read_gosa(1))
PY
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_stencil_tb2 -s 0 -c 1 \
  -o $OUT/m_flow python /tmp/mflow.py M 20 > $OUT/ncu_m.log 2>&1
tail -2 $OUT/ncu_m.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_stencil_tb2 -s 1 -c 1 \
  -o $OUT/l_tb2 python /tmp/mflow.py L 4 > $OUT/ncu_l.log 2>&1
tail -2 $OUT/ncu_l.log
