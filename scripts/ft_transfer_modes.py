"""Transfer-hoisting ablation on NAS FT through the generated executor (the paper's
batched transfers, on the second application).

For each class, the pattern with every exact loop on the B200 (tests/test_generic.py
_ft_exact_ids) runs with transfer_mode="batched" (Planner.plan: hoisted, batched,
temp regions) and "per-loop" (plan_transfers: one region per kernel); output verified
against NPB's checksums.  One JSON line per (class, mode).

    python scripts/ft_transfer_modes.py [S W A]
"""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

from paper_2002_12115_b200 import generic  # noqa: E402
from paper_2002_12115_b200.apps import ft  # noqa: E402
from test_generic import _ft_exact_ids  # noqa: E402


def main():
    for cls in sys.argv[1:] or ["S", "W", "A"]:
        prog = ft.program(cls)
        exact = _ft_exact_ids(prog)
        for mode in ("batched", "per-loop"):
            with generic.GenEvaluator(f"ft_{cls.lower()}", devices=[0], transfer_mode=mode) as ev:
                g = tuple(int(l in exact) for l in ev.eligible_ids)
                ts = [ev.measure(g).seconds for _ in range(3)]
                st = ev.stats[g]
                print(json.dumps({
                    "class": cls, "mode": mode, "ms": [round(t * 1e3, 2) for t in ts],
                    "plan_entries": len(ev.plan(g).entries),
                    "h2d_MB": st["h2d_bytes"] / 1e6, "d2h_MB": st["d2h_bytes"] / 1e6,
                    "n_h2d": st["n_h2d"], "n_d2h": st["n_d2h"], "launches": st["n_launch"],
                    "checksum_err": ft.checksum_error(ev.outputs[g], cls)}), flush=True)


if __name__ == "__main__":
    main()
