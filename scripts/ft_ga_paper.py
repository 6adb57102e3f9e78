"""NAS FT with the paper's GA setting on the B200.

PAPER.md:179-183, 226: NAS.FT, 65 genes, population 30, 20 generations, Pc 0.9,
Pm 0.05, elitism; reported 10.0x over all-CPU.  Here: class S (and W) through the
generated executor (generic.GenEvaluator), nested genes under their outermost anchor,
every run's output verified against the all-CPU program; gene sets "verified" (loops
whose device version the execution probe verified: 64 of 79 at S -- the paper's 65)
and "screened" (verified and not slower alone than all-CPU, the paper's narrowing).
Reported against the all-CPU program and the exact pattern (every verified FFT/bulk
loop on the device: tests/test_generic.py FT_EXACT).

    python scripts/ft_ga_paper.py [--apps ft_s,ft_w] [--seeds 0,1,2] [--out ...]
"""
import argparse
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2002_12115_b200 import ga, generic  # noqa: E402

FT_EXACT_S = [0, 3, 4, 10, 13, 16, 19, 22, 25, 28, 31, 34, 37, 40, 43, 45, 49, 53, 56, 59,
              62, 65, 68, 71, 74, 77, 80, 83, 86, 88, 91]


def main():
    ap = argparse.ArgumentParser(description=__doc__.splitlines()[0])
    ap.add_argument("--apps", default="ft_s")
    ap.add_argument("--genes", default="verified,screened")
    ap.add_argument("--seeds", default="0,1,2")
    ap.add_argument("--pop", type=int, default=30)
    ap.add_argument("--gens", type=int, default=20)
    ap.add_argument("--workers", type=int, default=4)
    ap.add_argument("--out", default=str(ROOT / "profiles" / "r02_ft_ga_paper.jsonl"))
    a = ap.parse_args()
    out = open(a.out, "w")
    for app in a.apps.split(","):
        for genes in a.genes.split(","):
            t0 = time.perf_counter()
            with generic.GenEvaluator(app, devices=[0], workers_per_device=a.workers,
                                      verify_each=True, nested_policy="outermost",
                                      genes=genes) as ev:
                probe_s = time.perf_counter() - t0
                ev.prepare()
                cpu_s = min(ev.measure((0,) * ev.gene_length).seconds for _ in range(3))
                exact_s = None
                if app == "ft_s" and set(FT_EXACT_S) <= set(ev.eligible_ids):
                    g = tuple(int(l in FT_EXACT_S) for l in ev.eligible_ids)
                    exact_s = min(ev.measure(g).seconds for _ in range(3))
                for seed in (int(s) for s in a.seeds.split(",")):
                    t1 = time.perf_counter()
                    res = ga.run_ga(ga.GAConfig(population=a.pop, generations=a.gens,
                                                rng_seed=seed), ev.gene_length, ev)
                    wall = time.perf_counter() - t1
                    b = res.best
                    best_s = min(ev.measure(b.genome).seconds for _ in range(3))
                    row = {"app": app, "genes": genes, "gene_length": ev.gene_length,
                           "population": a.pop, "generations": a.gens, "seed": seed,
                           "probe_s": probe_s, "ga_wall_s": wall, "evaluations": res.evaluations,
                           "evals_per_s": res.evaluations / wall,
                           "all_cpu_s": cpu_s, "exact_pattern_s": exact_s,
                           "best_time_s": best_s, "speedup_vs_all_cpu": cpu_s / best_s,
                           "exact_speedup": (cpu_s / exact_s) if exact_s else None,
                           "best_loops_on_device": [l for l, x in zip(ev.eligible_ids, b.genome)
                                                    if x],
                           "per_generation_best_s": [r.best_time_s for r in res.records]}
                    out.write(json.dumps(row) + "\n")
                    out.flush()
                    print(json.dumps({k: v for k, v in row.items()
                                      if k not in ("per_generation_best_s",
                                                   "best_loops_on_device")}), flush=True)
    out.close()


if __name__ == "__main__":
    main()
