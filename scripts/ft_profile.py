"""Run NAS FT's exact pattern (every exact FFT/bulk loop on the device) twice; the
second run inside an NVTX range "ft_exact" so ncu can capture just its kernels:

    ncu --nvtx --nvtx-include "ft_exact/" --metrics gpu__time_duration.sum,\
dram__bytes_read.sum,dram__bytes_write.sum --csv --log-file out.csv \
        python scripts/ft_profile.py A
"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import torch  # noqa: E402  (NVTX)

from paper_2002_12115_b200 import generic  # noqa: E402
from paper_2002_12115_b200.apps import ft  # noqa: E402
from test_generic import _ft_exact_ids  # noqa: E402


def main():
    cls = sys.argv[1] if len(sys.argv) > 1 else "S"
    prog = ft.program(cls)
    exact = _ft_exact_ids(prog)
    # long watchdog: under ncu every launch of the profiled run is replayed
    with generic.GenEvaluator(f"ft_{cls.lower()}", devices=[0], timeout_s=3000.0) as ev:
        g = tuple(int(l in exact) for l in ev.eligible_ids)
        m = ev.measure(g)
        print("warm-up run:", m, flush=True)
        torch.cuda.nvtx.range_push("ft_exact")
        m = ev.measure(g)
        torch.cuda.nvtx.range_pop()
        st = ev.stats[g]
        if m.seconds is None:
            raise SystemExit(f"exact pattern did not run: {m} {st}")
        print(f"ft_{cls.lower()} exact: {m.seconds * 1e3:.1f} ms, {st['n_launch']} launches, "
              f"checksum error {ft.checksum_error(ev.outputs[g], cls):.1e}")


if __name__ == "__main__":
    main()
