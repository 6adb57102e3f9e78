#!/bin/bash
TAG=${1:-ncu_tb2}
OUT=gpurun_out/$TAG
mkdir -p $OUT
cat > /tmp/tb2run.py <<'PY'
import sys; sys.path.insert(0,'.')
from paper_2002_12115_b200 import native as N
from paper_2002_12115_b200.apps import himeno
lib=N.load(); lib.hp_set_temporal_blocking(1)
sz=himeno.size('L')
with N.Context(0, sz.I, sz.J, sz.K) as c:
    c.init_device(); c.jacobi_device(6,1)
PY
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_stencil_tb2 -s 1 -c 1 \
  -o $OUT/tb2 python /tmp/tb2run.py > $OUT/ncu.log 2>&1
tail -2 $OUT/ncu.log
