#!/bin/bash
TAG=${1:-promo}
OUT=gpurun_out/$TAG
mkdir -p $OUT
for pr in "2,2,0,0" "2,2,2,2" "0,0,0,0" "2,0,0,2" "1,1,1,1"; do
  for tb in 0 1; do
    HIMENO_TMA_PROMO=$pr HIMENO_TB=$tb timeout 120 python -c "
import sys; sys.path.insert(0,'.')
from paper_2002_12115_b200 import native as N
from paper_2002_12115_b200.apps import himeno
lib=N.load(); lib.hp_set_temporal_blocking($tb)
for name in ('L','M'):
    sz=himeno.size(name)
    with N.Context(0, sz.I, sz.J, sz.K) as c:
        c.init_device(); c.jacobi_device(4,1)
        best=min((c.time_jacobi(10,1) for _ in range(3)), key=lambda k: k.stencil_ms)
        print('promo $pr tb $tb', name, 'pass_ms %.4f iters %.1f GBs %.0f GFLOPs %.0f' % (best.stencil_ms, best.stencil_iters, 56*sz.interior_points/best.stencil_ms/1e6, 34*sz.interior_points*best.stencil_iters/best.stencil_ms/1e6))
" 2>&1 | tail -2
  done
done
