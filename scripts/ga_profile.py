"""Where does a GA generation's wall time go?  Per-measure breakdown on one GPU.

Runs run_ga (M, nn=3, pop 20 x gen 10, seed 0) through B200Evaluator with the
evaluator's pieces timed: lowering (plan + schedule, Python), hp_run total and
the program wall time inside it (the rest of hp_run is the fresh-process reset),
and the time run_ga spends outside measure.  Prints one JSON line per measure
and a summary line.
"""
import argparse
import json
import sys
import threading
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2002_12115_b200 import ga  # noqa: E402
from paper_2002_12115_b200.evaluator import B200Evaluator  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--size", default="M")
    ap.add_argument("--nn", type=int, default=3)
    ap.add_argument("--pop", type=int, default=20)
    ap.add_argument("--gens", type=int, default=10)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--workers", type=int, default=4)
    ap.add_argument("--quiet", action="store_true")
    a = ap.parse_args()
    rows, lock = [], threading.Lock()
    with B200Evaluator(a.size, nn=a.nn, devices=[0], workers_per_device=a.workers) as ev:
        ev.prepare()
        ev.measure((0,) * ev.gene_length)
        orig_lowered, orig_execute = ev.lowered, ev._execute

        def execute(genome):
            t0 = time.perf_counter()
            low = orig_lowered(genome)
            t1 = time.perf_counter()
            if low.failure is not None:
                with lock:
                    rows.append({"g": ga.genome_str(genome), "lower_ms": (t1 - t0) * 1e3,
                                 "failed": True, "t": t0})
                return low, None, None
            slot = ev._free.get()
            try:
                t2 = time.perf_counter()
                res = ev._context(slot).run(low.schedule)
                t3 = time.perf_counter()
            finally:
                ev._free.put(slot)
            with lock:
                rows.append({"g": ga.genome_str(genome), "lower_ms": (t1 - t0) * 1e3,
                             "wait_ms": (t2 - t1) * 1e3, "hp_run_ms": (t3 - t2) * 1e3,
                             "wall_ms": res.wall_s * 1e3, "t": t0, "slot": slot})
            return low, res, slot

        ev._execute = execute
        t0 = time.perf_counter()
        res = ga.run_ga(ga.GAConfig(population=a.pop, generations=a.gens, rng_seed=a.seed),
                        ev.gene_length, ev)
        el = time.perf_counter() - t0
    if not a.quiet:
        for r in rows:
            r["t"] -= t0
            print(json.dumps(r))
    ok = [r for r in rows if not r.get("failed")]
    summ = {
        "wall_s": el, "evals": res.evaluations, "valid": len(ok),
        "evals_per_s": res.evaluations / el, "gens_per_s": a.gens / el,
        "sum_lower_ms": sum(r["lower_ms"] for r in rows),
        "sum_hp_run_ms": sum(r["hp_run_ms"] for r in ok),
        "sum_prog_wall_ms": sum(r["wall_ms"] for r in ok),
        "sum_reset_ms": sum(r["hp_run_ms"] - r["wall_ms"] for r in ok),
        "max_prog_wall_ms": max((r["wall_ms"] for r in ok), default=0.0),
        "best": ga.genome_str(res.best.genome), "best_ms": res.best.time_s * 1e3,
    }
    print(json.dumps(summ))


if __name__ == "__main__":
    main()
