#!/bin/bash
# Two-step kernel tile shapes (HIMENO_TB2_SHAPE 0..3, see stencil_tma.cu): bit-exactness
# (temporal-blocking, headline, slab and ragged-grid tests) and pass times per grid.
TAG=${1:-tb2shape}
SHAPES=${2:-"0 1 2 3"}
OUT=gpurun_out/$TAG
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
for sh in $SHAPES; do
  HIMENO_TB2_SHAPE=$sh timeout 900 python -m pytest tests -m gpu -q -x \
    -k "temporal or headline or group or tiny or zero_iterations or device_jacobi" > $OUT/pytest_s$sh.log 2>&1
  echo "shape=$sh pytest rc=$?" >> $OUT/pytest_s$sh.log
  tail -2 $OUT/pytest_s$sh.log
  for ch in 32 64; do
  HIMENO_TB2_CHUNK=$ch HIMENO_TB2_SHAPE=$sh timeout 180 python -c "
import sys; sys.path.insert(0,'.')
from paper_2002_12115_b200 import native as N
from paper_2002_12115_b200.apps import himeno
lib=N.load(); lib.hp_set_temporal_blocking(1)
for name in ('L','M','XL'):
    sz=himeno.size(name)
    with N.Context(0, sz.I, sz.J, sz.K) as c:
        c.init_device(); c.jacobi_device(4,1)
        best=min((c.time_jacobi(10,1) for _ in range(5)), key=lambda k: k.stencil_ms)
        it=best.stencil_iters
        print('shape $sh chunk $ch', name, 'pass_ms %.4f iters %.1f GBs %.0f GFLOPs %.0f' % (best.stencil_ms, it, 56*sz.interior_points/best.stencil_ms/1e6, 34*sz.interior_points*it/best.stencil_ms/1e6))
" 2>&1 | tail -3
  done
done
