"""Fit the reference-format cost model to B200 measurements; compare optima.

    python scripts/calibrate_costmodel.py profiles/r01_evalall_M.jsonl [--out profiles/...json]

Bandwidth and latency of a transfer event come from the measured runs (total
bytes moved / host time blocked in transfers; 10 us per event); the loop terms
are fitted (costmodel.calibrate).  Reports fit residual, rank correlation of
predicted vs measured fitness over the runnable genomes, and whether the
surrogate's optimum is the measured optimum.
"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2002_12115_b200 import costmodel as cm  # noqa: E402
from paper_2002_12115_b200.apps import himeno  # noqa: E402
from paper_2002_12115_b200.ga import genome_str  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("measurements")
    ap.add_argument("--out")
    ap.add_argument("--latency", type=float, default=1e-5)
    ap.add_argument("--bandwidth", type=float,
                    help="bytes/s of a transfer event when the table has no transfer stats "
                         "(e.g. 2.075e10, measured in profiles/r01_evalall_M.jsonl)")
    args = ap.parse_args()
    prog = himeno.program()
    loops, refs, elig = prog.model.loops, prog.model.refs, list(prog.eligible)
    rows = [json.loads(l) for l in Path(args.measurements).read_text().splitlines()]
    rows = [r for r in rows if not r.get("summary") and r.get("time_s")]
    moved = sum((r.get("h2d_bytes") or 0) + (r.get("d2h_bytes") or 0) for r in rows)
    blocked = sum(r.get("xfer_s") or 0 for r in rows)
    bw = moved / blocked if blocked > 0 else (args.bandwidth or 2.5e10)
    samples = [(tuple(int(c) for c in r["genome"]), float(r["time_s"])) for r in rows]
    meas = [t for _, t in samples]
    best_meas = min(samples, key=lambda s: s[1])
    doc = {"measurements": args.measurements, "samples": len(samples),
           "bandwidth_bytes_per_s": bw, "latency_s": args.latency,
           "measured_optimum": [genome_str(best_meas[0]), best_meas[1]]}
    for name, nest in (("additive", False), ("nest_aware", True)):
        cal = cm.calibrate(samples, loops, refs, elig, bw, args.latency, nest_aware=nest)
        ev = cm.CostModelEvaluator(cal.model, loops, refs, elig, nest_aware=nest)
        pred = [ev.measure(g).seconds for g, _ in samples]
        best_pred, t_pred = cm.optimum_over(cal.model, loops, refs, elig,
                                            [g for g, _ in samples], nest_aware=nest)
        meas_of_pred = dict(samples)[best_pred]
        doc[name] = {"residual_rms_s": cal.residual_rms_s, "spearman": cm.spearman(pred, meas),
                     "surrogate_optimum": [genome_str(best_pred), t_pred, meas_of_pred],
                     "surrogate_optimum_regret": meas_of_pred / best_meas[1] - 1.0,
                     "model": cal.model.to_json()}
    text = json.dumps(doc, indent=1)
    if args.out:
        Path(args.out).write_text(text + "\n")
    print(json.dumps({k: ({kk: vv for kk, vv in v.items() if kk != "model"}
                          if isinstance(v, dict) else v) for k, v in doc.items()}, indent=1))


if __name__ == "__main__":
    main()
