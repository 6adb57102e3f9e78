"""Time every tuned-stencil configuration (hp_set_stencil_config) on one grid.

    python scripts/sweep_stencil.py [--size L] [--nn 10] [--reps 5]

Prints one JSON line per configuration: mean stencil launch ms (CUDA events,
best of reps), achieved GB/s at 56 B/pt, and the gosa after a fixed number of
iterations (all configurations must agree bit-for-bit on p; gosa to 1e-12).
"""
import argparse
import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2002_12115_b200 import native as N  # noqa: E402
from paper_2002_12115_b200.apps import himeno  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--size", default="L")
    ap.add_argument("--nn", type=int, default=10)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--variant", type=int, default=1)
    args = ap.parse_args()
    sz = himeno.size(args.size)
    lib = N.load()
    ncfg = lib.hp_set_stencil_config(0)
    ref_p = None
    with N.Context(0, sz.I, sz.J, sz.K) as ctx:
        for cfg in range(ncfg):
            lib.hp_set_stencil_config(cfg)
            ctx.init_device()
            ctx.jacobi_device(3, args.variant)
            gosa = ctx.read_gosa(1)
            p = ctx.read_field("p", 1)
            same = True if ref_p is None else bool(np.array_equal(p, ref_p))
            ref_p = p if ref_p is None else ref_p
            best = None
            for _ in range(args.reps):
                kt = ctx.time_jacobi(args.nn, args.variant)
                best = kt if best is None or kt.stencil_ms < best.stencil_ms else best
            gbs = 56 * sz.interior_points / (best.stencil_ms / 1e3) / 1e9
            print(json.dumps({"cfg": cfg, "size": sz.name, "stencil_ms": best.stencil_ms,
                              "gbs": gbs, "other_ms": best.other_ms, "total_ms": best.total_ms,
                              "gosa": gosa, "p_same_as_cfg0": same}), flush=True)
        lib.hp_set_stencil_config(7)


if __name__ == "__main__":
    main()
