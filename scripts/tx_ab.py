"""A/B of the two-step kernels on one B200: k_stencil_tx (tile exchange) vs
k_stencil_tb2 (halo recompute), alternating runs.  Prints one line per run:
grid, kernel, per-pass ms (CUDA events), GFLOP/s of a jacobi(nn) step."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2002_12115_b200 import native as N  # noqa: E402
from paper_2002_12115_b200.apps import himeno  # noqa: E402

grids = sys.argv[1].split(",") if len(sys.argv) > 1 else ["M", "L"]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
nn = 100
for name in grids:
    sz = himeno.size(name)
    nint = (sz.I - 3) * (sz.J - 3) * (sz.K - 3)
    with N.Context(0, sz.I, sz.J, sz.K) as ctx:
        ctx.init_device()
        for r in range(reps):
            for mode in ("1", "0"):
                os.environ["HIMENO_TX"] = mode
                ctx.time_steps(2, nn, 1)
                kern = N.last_two_step_kernel()
                ms = ctx.time_steps(5, nn, 1) / 5
                kt = ctx.time_jacobi(nn, 1)
                gf = 34.0 * nint * nn / (ms * 1e-3) / 1e9
                gbs = 56.0 * nint / (kt.stencil_ms * 1e-3) / 1e9
                print(f"{name} {kern:14s} pass_ms {kt.stencil_ms:.4f} step_ms {ms:.3f} "
                      f"GFLOPs {gf:.0f} pass_GBs {gbs:.0f} tx_status {ctx.tx_status()}", flush=True)
