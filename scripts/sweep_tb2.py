"""Sweep the two-step kernel's tile shape x planes-per-unit on L, M, XL (one process).

    python scripts/sweep_tb2.py > profiles/r01_tb2_shapes.txt

HIMENO_TB2_SHAPE / HIMENO_TB2_CHUNK are read per launch (stencil_tma.cu tb2_choose), so
they are set here between timings; the last line per grid is the automatic choice.
"""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2002_12115_b200 import native as N  # noqa: E402
from paper_2002_12115_b200.apps import himeno  # noqa: E402

CHUNKS = (24, 32, 40, 48, 64, 88, 96, 128)
SHAPES = [int(x) for x in os.environ.get("SWEEP_SHAPES", "0,1,2,3,4").split(",")]


def timed(ctx, sz):
    best = min((ctx.time_jacobi(10, 1) for _ in range(3)), key=lambda k: k.stencil_ms)
    return best.stencil_ms, 34 * sz.interior_points * best.stencil_iters / best.stencil_ms / 1e6


def main():
    lib = N.load()
    lib.hp_set_temporal_blocking(1)
    for name in sys.argv[1:] or ("L", "M", "XL"):
        sz = himeno.size(name)
        with N.Context(0, sz.I, sz.J, sz.K) as c:
            c.init_device()
            c.jacobi_device(4, 1)
            for shape in SHAPES:
                for ch in CHUNKS:
                    os.environ["HIMENO_TB2_SHAPE"] = str(shape)
                    os.environ["HIMENO_TB2_CHUNK"] = str(ch)
                    ms, gf = timed(c, sz)
                    print(f"{name} shape {shape} chunk {ch:3d} pass_ms {ms:.4f} GFLOPs {gf:.0f}", flush=True)
            os.environ.pop("HIMENO_TB2_SHAPE")
            os.environ.pop("HIMENO_TB2_CHUNK")
            ms, gf = timed(c, sz)
            print(f"{name} auto pass_ms {ms:.4f} GFLOPs {gf:.0f}", flush=True)


if __name__ == "__main__":
    main()
