#!/bin/bash
for ch in 24 32 48 64 96; do
  HIMENO_CHUNK=$ch timeout 120 python -c "
import sys; sys.path.insert(0,'.')
from paper_2002_12115_b200 import native as N
from paper_2002_12115_b200.apps import himeno
lib=N.load(); lib.hp_set_temporal_blocking(1)
for name in ('L','M','XL'):
    sz=himeno.size(name)
    with N.Context(0, sz.I, sz.J, sz.K) as c:
        c.init_device(); c.jacobi_device(4,1)
        best=min((c.time_jacobi(10,1) for _ in range(3)), key=lambda k: k.stencil_ms)
        it=best.stencil_iters
        print('chunk $ch', name, 'pass_ms %.4f GFLOPs %.0f' % (best.stencil_ms, 34*sz.interior_points*it/best.stencil_ms/1e6))
" 2>&1 | tail -3
done
