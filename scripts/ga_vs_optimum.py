"""Does the GA find the optimum?  SPEC acceptance 1 on real B200 measurements.

The reference's brute_force_optimum (acctuner/evaluators.py:131-147) enumerates every
genome with a (cost-model) evaluator; SPEC.md:552 asks that the GA land within 5 % of
that optimum.  Here the evaluator is the B200 itself (Himeno M, nn = 3):

  A  every runnable genome (the 272 without nested gene=1 loops) measured on the GPU,
     best of `--reps` runs -> the fitness table and its optimum;
  B  run_ga replayed against that table for seeds 0..9, population x generations
     10 x 10 (the paper's M = 10, T = 10 for Himeno) and 20 x 20
     (BASELINE config 4); nested genomes fail (penalty) as the reference's OpenACC
     compile does.  The replay is deterministic: this repo's run_ga equals the
     reference's for the same fitness table (tests/test_ga.py,
     tests/test_reference_driver.py);
  C  the same GA runs live on the GPU (B200Evaluator, 4 worker slots), with nested genes
     rejected ("reject") and with nested genes running their outermost anchor
     ("outermost"); the genome found is scored by its table time (the live timings of one
     run are noisy), and the live best is re-measured against the optimum.

    python scripts/ga_vs_optimum.py [--out profiles/r02_ga_vs_optimum.json]

Phase B alone (no GPU) with --table <jsonl from phase A>.
"""
import argparse
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2002_12115_b200 import ga  # noqa: E402
from paper_2002_12115_b200.evaluator import MeasuredTime, valid_genomes  # noqa: E402

CONFIGS = ((10, 10), (20, 20))
SEEDS = tuple(range(10))
WITHIN = 0.05


class Replay:
    """Fitness table evaluator: runnable genomes -> their measured time, others fail."""

    max_concurrency = 1
    deterministic = True

    def __init__(self, table: dict):
        self.table = table

    def measure(self, genome):
        t = self.table.get(tuple(genome))
        if t is None:
            return MeasuredTime.failed("nested compute construct")
        return MeasuredTime.ok(t)


def measure_table(size: str, nn: int, reps: int, host_build: str = "tuned") -> dict:
    from paper_2002_12115_b200.evaluator import B200Evaluator
    table = {}
    with B200Evaluator(size, nn=nn, host_build=host_build) as ev:
        ev.measure((0,) * ev.gene_length)
        for g in valid_genomes(ev.loops, ev.eligible_ids):
            ts = [ev.measure(g).seconds for _ in range(reps)]
            table[g] = min(t for t in ts if t)
    return table


def replay_sweep(table: dict, gene_len: int = 13) -> list:
    opt_g = min(table, key=table.get)
    opt = table[opt_g]
    rows = []
    for pop, gens in CONFIGS:
        for seed in SEEDS:
            res = ga.run_ga(ga.GAConfig(population=pop, generations=gens, rng_seed=seed),
                            gene_len, Replay(table))
            b = res.best
            rows.append({"phase": "replay", "population": pop, "generations": gens, "seed": seed,
                         "best_genome": ga.genome_str(b.genome), "best_time_s": b.time_s,
                         "ratio_to_optimum": b.time_s / opt if b.time_s < 1000 else None,
                         "evaluations": res.evaluations,
                         "runnable_evaluated": sum(1 for r in res.records for i in r.individuals
                                                   if i.eval_source == "fresh"),
                         "within_5pct": b.time_s <= (1 + WITHIN) * opt})
    return rows


def live_sweep(table: dict, size: str, nn: int, workers: int, host_build: str = "tuned") -> list:
    from paper_2002_12115_b200.evaluator import B200Evaluator
    opt_g = min(table, key=table.get)
    rows = []
    for policy in ("reject", "outermost"):
        with B200Evaluator(size, nn=nn, workers_per_device=workers, nested_policy=policy,
                           host_build=host_build) as ev:
            ev.prepare()
            ev.measure((0,) * ev.gene_length)
            for pop, gens in CONFIGS:
                for seed in SEEDS:
                    t0 = time.perf_counter()
                    res = ga.run_ga(ga.GAConfig(population=pop, generations=gens, rng_seed=seed),
                                    ev.gene_length, ev)
                    wall = time.perf_counter() - t0
                    b = res.best
                    row = {"phase": "live", "nested_policy": policy, "population": pop,
                           "generations": gens, "seed": seed,
                           "best_genome": ga.genome_str(b.genome), "best_time_s": b.time_s,
                           "wall_s": wall, "evaluations": res.evaluations}
                    if b.time_s < 1000:
                        # the effective pattern under "outermost" is the genome with its
                        # inner genes cleared; score it by the table, and re-measure both
                        eff = ev.lowered(b.genome).loop_kind
                        t_best = min(ev.measure(b.genome).seconds for _ in range(5))
                        t_opt = min(ev.measure(opt_g).seconds for _ in range(5))
                        row.update(remeasured_best_s=t_best, remeasured_optimum_s=t_opt,
                                   ratio_to_optimum=t_best / t_opt,
                                   within_5pct=t_best <= (1 + WITHIN) * t_opt,
                                   effective_kinds=list(eff) if eff is not None else None)
                        if tuple(b.genome) in table:
                            row["table_ratio"] = table[tuple(b.genome)] / table[opt_g]
                    else:
                        row.update(ratio_to_optimum=None, within_5pct=False)
                    rows.append(row)
                    print(json.dumps(row), file=sys.stderr, flush=True)
    return rows


def summarize(rows: list) -> list:
    out = []
    keys = sorted({(r["phase"], r.get("nested_policy", "reject"), r["population"],
                    r["generations"]) for r in rows})
    for phase, pol, pop, gens in keys:
        sel = [r for r in rows if r["phase"] == phase and r.get("nested_policy", "reject") == pol
               and r["population"] == pop and r["generations"] == gens]
        ratios = [r["ratio_to_optimum"] for r in sel
                  if r.get("ratio_to_optimum") and r["best_time_s"] < 1000]
        out.append({"phase": phase, "nested_policy": pol, "population": pop, "generations": gens,
                    "seeds": len(sel), "within_5pct": sum(1 for r in sel if r["within_5pct"]),
                    "found_runnable": len(ratios),
                    "median_ratio": sorted(ratios)[len(ratios) // 2] if ratios else None,
                    "worst_ratio": max(ratios) if ratios else None})
    return out


def main():
    ap = argparse.ArgumentParser(description=__doc__.splitlines()[0])
    ap.add_argument("--size", default="M")
    ap.add_argument("--nn", type=int, default=3)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--workers", type=int, default=4)
    ap.add_argument("--table", help="JSONL table (genome, time_s): skip phase A")
    ap.add_argument("--table-out", default=str(ROOT / "profiles" / "r02_evalall_M.jsonl"))
    ap.add_argument("--no-live", action="store_true")
    ap.add_argument("--host-build", default="tuned", choices=["tuned", "reference"],
                    help="gene-0 loops: tuned host build or the reference's gcc -O2 template")
    ap.add_argument("--out", default=str(ROOT / "profiles" / "r02_ga_vs_optimum.json"))
    a = ap.parse_args()
    if a.table:
        table = {}
        for line in open(a.table):
            d = json.loads(line)
            if "genome" in d and d.get("time_s"):
                table[tuple(int(c) for c in d["genome"])] = d["time_s"]
    else:
        table = measure_table(a.size, a.nn, a.reps, a.host_build)
        with open(a.table_out, "w") as fh:
            for g, t in sorted(table.items(), key=lambda kv: kv[1]):
                fh.write(json.dumps({"genome": ga.genome_str(g), "time_s": t}) + "\n")
    opt_g = min(table, key=table.get)
    rows = replay_sweep(table)
    if not a.no_live:
        rows += live_sweep(table, a.size, a.nn, a.workers, a.host_build)
    doc = {"size": a.size, "nn": a.nn, "host_build": a.host_build, "runnable_genomes": len(table),
           "optimum": {"genome": ga.genome_str(opt_g), "time_s": table[opt_g]},
           "criterion": "best within 5 % of the optimum (SPEC.md:552)",
           "summary": summarize(rows), "runs": rows}
    Path(a.out).write_text(json.dumps(doc, indent=1) + "\n")
    print(json.dumps(doc["summary"], indent=1))


if __name__ == "__main__":
    main()
