"""Evaluate every valid (non-nested) genome once on one GPU; per-genome stats.

    python scripts/eval_all.py [--size M] [--nn 3] [--mode batched|per-loop] [--timeout 60]

One JSON line per genome (time, transfers, launches) sorted by time, then a
summary line with the optimum -- the real-evaluator analogue of the reference's
brute_force_optimum (evaluators.py:131-147) over the 272 runnable patterns.
"""
import argparse
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2002_12115_b200.evaluator import B200Evaluator, valid_genomes  # noqa: E402
from paper_2002_12115_b200.ga import genome_str  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--size", default="M")
    ap.add_argument("--nn", type=int, default=3)
    ap.add_argument("--mode", default="batched")
    ap.add_argument("--timeout", type=float, default=60.0)
    ap.add_argument("--limit", type=int, default=0)
    args = ap.parse_args()
    rows = []
    t0 = time.perf_counter()
    with B200Evaluator(args.size, nn=args.nn, transfer_mode=args.mode,
                       timeout_s=args.timeout) as ev:
        ev.measure((0,) * ev.gene_length)
        genomes = valid_genomes(ev.loops, ev.eligible_ids)
        if args.limit:
            genomes = genomes[:args.limit]
        for g in genomes:
            m = ev.measure(g)
            st = ev.stats.get(g, {})
            rows.append({"genome": genome_str(g), "time_s": m.seconds,
                         "timed_out": m.timed_out, "failure": m.failure,
                         **{k: st.get(k) for k in ("h2d_bytes", "d2h_bytes", "n_h2d", "n_d2h",
                                                   "n_implicit", "n_skipped_stale", "n_launch",
                                                   "host_s", "xfer_s")}})
            print(json.dumps(rows[-1]), file=sys.stderr, flush=True)
    ok = [r for r in rows if r["time_s"]]
    ok.sort(key=lambda r: r["time_s"])
    for r in ok:
        print(json.dumps(r))
    print(json.dumps({"summary": True, "size": args.size, "nn": args.nn, "mode": args.mode,
                      "evaluated": len(rows), "ok": len(ok), "wall_s": time.perf_counter() - t0,
                      "best": ok[0] if ok else None, "worst": ok[-1] if ok else None}))


if __name__ == "__main__":
    main()
