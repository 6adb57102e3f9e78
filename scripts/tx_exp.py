"""Exchange-kernel experiments on L: per-pass time under env settings given as
NAME=VALUE[,NAME=VALUE] arguments (each argument is one configuration)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2002_12115_b200 import native as N  # noqa: E402
from paper_2002_12115_b200.apps import himeno  # noqa: E402

grid = os.environ.get("GRID", "L")
sz = himeno.size(grid)
nint = (sz.I - 3) * (sz.J - 3) * (sz.K - 3)
confs = sys.argv[1:] or [""]
with N.Context(0, sz.I, sz.J, sz.K) as ctx:
    ctx.init_device()
    for rep in range(2):
        for conf in confs:
            saved = {}
            for kv in filter(None, conf.split(",")):
                k, v = kv.split("=")
                saved[k] = os.environ.get(k)
                os.environ[k] = v
            ctx.time_steps(1, 20, 1)
            kt = ctx.time_jacobi(40, 1)
            print(f"{grid} {conf or 'default':40s} {N.last_two_step_kernel():14s} pass_ms {kt.stencil_ms:.4f} "
                  f"GBs {56.0 * nint / (kt.stencil_ms * 1e-3) / 1e9:.0f}", flush=True)
            for k, v in saved.items():
                if v is None:
                    os.environ.pop(k, None)
                else:
                    os.environ[k] = v
