"""Per-pass time of one rank's slab of L (BASELINE config 3 at 2/4/8 GPUs), two-step
kernels compared on one GPU: k_stencil_tb2 vs k_stencil_tx (HIMENO_TX=1), CUDA events per
pass, no exchange (hp_time_jacobi on the slab context)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2002_12115_b200 import dd, native as N  # noqa: E402
from paper_2002_12115_b200.apps import himeno  # noqa: E402

sz = himeno.size("L")
for ranks in (1, 2, 4, 8):
    r = min(1, ranks - 1)
    b, e = dd.slab_range(sz.I, ranks, r) if ranks > 1 else (1, sz.I - 2)
    with N.Context(0, sz.I, sz.J, sz.K, slab=(b, e) if ranks > 1 else None) as c:
        c.init_device()
        pts = (e - b) * (sz.J - 3) * (sz.K - 3)
        for rep in range(2):
            for tx in ("0", "1"):
                os.environ["HIMENO_TX"] = tx
                c.time_jacobi(8, 1)
                kt = c.time_jacobi(40, 1)
                print(f"L/{ranks} planes {e - b:3d} {N.last_two_step_kernel():14s} pass_us "
                      f"{kt.stencil_ms * 1e3:8.2f}  GB/s {56.0 * pts / (kt.stencil_ms * 1e-3) / 1e9:6.0f}",
                      flush=True)
