"""BASELINE config 5 on one GPU: batched (Planner.plan) vs per-loop (raw plan_transfers +
implicit per-kernel copies) transfer plans on the same genomes.

    python scripts/transfer_modes.py [--size XL] [--nn 3] [--repeats 3]

For each genome and mode: best-of-`repeats` fitness time (the evaluator's wall clock,
evaluators.py:207-214 semantics), dynamic H2D/D2H bytes and copy counts, implicit
copies, stale updates skipped, kernel launches, and the stdout digest (gosa + p
samples) to show both modes compute the same program.  One JSON line per
(genome, mode), then a summary line.
"""
import argparse
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2002_12115_b200.evaluator import B200Evaluator  # noqa: E402
from paper_2002_12115_b200.ga import genome_str  # noqa: E402

# GPU-heavy patterns (all-CPU patterns at XL take minutes of host time per run)
GENOMES = ["1001001000000",   # init + device time loop (M optimum)
           "1001000100100",   # init + stencil + copy nests
           "0000001000000",   # device time loop only
           "0000000100100",   # stencil + copy nests (BASELINE config 2 default)
           "1001000100000",   # stencil on device, copy on host
           "0001000100100"]   # init nest A on host


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--size", default="XL")
    ap.add_argument("--nn", type=int, default=3)
    ap.add_argument("--repeats", type=int, default=3)
    ap.add_argument("--timeout", type=float, default=300.0)
    args = ap.parse_args()
    rows = []
    t0 = time.perf_counter()
    for mode in ("batched", "per-loop"):
        with B200Evaluator(args.size, nn=args.nn, transfer_mode=mode,
                           timeout_s=args.timeout) as ev:
            for gs in GENOMES:
                g = tuple(int(c) for c in gs)
                times = []
                m = None
                for _ in range(args.repeats):
                    m = ev.measure(g)
                    if m.seconds is None:
                        break
                    times.append(m.seconds)
                st = ev.stats.get(g, {})
                out = ev.run_for_output(g).split() if times else []
                plan = ev.plan(g)
                row = {"genome": genome_str(g), "mode": mode, "size": args.size, "nn": args.nn,
                       "time_s": min(times) if times else None,
                       "times_s": times, "failure": m.failure if m else None,
                       "plan_entries": len(plan.entries),
                       "gosa": out[0] if out else None,
                       "digest": out,
                       **{k: st.get(k) for k in ("h2d_bytes", "d2h_bytes", "n_h2d", "n_d2h",
                                                 "n_implicit", "n_skipped_stale", "n_launch",
                                                 "host_s", "xfer_s", "n_stale_reads")}}
                rows.append(row)
                print(json.dumps(row), flush=True)
    by = {(r["genome"], r["mode"]): r for r in rows}
    summary = []
    for gs in GENOMES:
        b, p = by.get((gs, "batched")), by.get((gs, "per-loop"))
        if b and p and b["time_s"] and p["time_s"]:
            summary.append({"genome": gs, "speedup_batched": p["time_s"] / b["time_s"],
                            "bytes_batched": b["h2d_bytes"] + b["d2h_bytes"],
                            "bytes_per_loop": p["h2d_bytes"] + p["d2h_bytes"],
                            "same_output": b["digest"] == p["digest"]})
    print(json.dumps({"summary": True, "size": args.size, "nn": args.nn,
                      "wall_s": time.perf_counter() - t0, "genomes": summary}))


if __name__ == "__main__":
    main()
