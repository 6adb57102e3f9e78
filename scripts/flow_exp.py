"""Device time loop jacobi(nn) per configuration (env NAME=VALUE[,...] per argument),
alternating, two rounds: ms per step, GFLOP/s, us per two-step pass."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2002_12115_b200 import native as N  # noqa: E402
from paper_2002_12115_b200.apps import himeno  # noqa: E402

grid = os.environ.get("GRID", "M")
nn = int(os.environ.get("NN", "100"))
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
            ctx.time_steps(2, nn, 1)
            ms = ctx.time_steps(5, nn, 1) / 5
            print(f"{grid} {conf or 'default':40s} {N.last_two_step_kernel():20s} step_ms {ms:.3f} "
                  f"GFLOPs {34.0 * nint * nn / (ms * 1e-3) / 1e9:.0f} us/pass {ms * 1e3 / (nn / 2):.2f}",
                  flush=True)
            for k, v in saved.items():
                if v is None:
                    os.environ.pop(k, None)
                else:
                    os.environ[k] = v
