#!/bin/bash
TAG=${1:-tb2}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 600 python -m pytest tests -m gpu -q -x -k "temporal or stencil_config or device_jacobi" > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
tail -2 $OUT/pytest_gpu.log
for tb in 0 1; do
  timeout 120 python -c "
import sys; sys.path.insert(0,'.')
from paper_2002_12115_b200 import native as N
from paper_2002_12115_b200.apps import himeno
lib=N.load(); lib.hp_set_temporal_blocking($tb)
for name in ('L','M','XL'):
    sz=himeno.size(name)
    with N.Context(0, sz.I, sz.J, sz.K) as c:
        c.init_device(); c.jacobi_device(4,1)
        best=min((c.time_jacobi(10,1) for _ in range(3)), key=lambda k: k.stencil_ms)
        it=best.stencil_iters
        print('tb $tb', name, 'pass_ms %.4f iters %.1f GBs %.0f GFLOPs %.0f' % (best.stencil_ms, it, 56*sz.interior_points/best.stencil_ms/1e6, 34*sz.interior_points*it/best.stencil_ms/1e6))
" 2>&1 | tail -3
done
