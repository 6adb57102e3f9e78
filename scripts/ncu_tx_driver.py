"""Small driver for ncu: L grid, one jacobi(4) (two two-step passes) on the default
two-step kernel (HIMENO_TX decides which), or k_stencil_tma<3> with HIMENO_SINGLE_STEP=1."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2002_12115_b200 import native as N  # noqa: E402
from paper_2002_12115_b200.apps import himeno  # noqa: E402

sz = himeno.size(sys.argv[1] if len(sys.argv) > 1 else "L")
if os.environ.get("HIMENO_SINGLE_STEP"):   # the one-iteration kernel k_stencil_tma<3>
    N.load().hp_set_temporal_blocking(0)
with N.Context(0, sz.I, sz.J, sz.K) as ctx:
    ctx.init_device()
    ctx.jacobi_device(4, 1)
    print(N.last_two_step_kernel(), ctx.read_gosa(1))
