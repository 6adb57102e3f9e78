import sys, os, json, time
sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..", "..")))
from paper_2002_12115_b200 import generic, ga
from paper_2002_12115_b200.apps import ft
app = sys.argv[1] if len(sys.argv) > 1 else "ft_s"
t0 = time.perf_counter()
ev = generic.GenEvaluator(app, devices=[0], workers_per_device=4, verify_each=True,
                          nested_policy="outermost", genes=sys.argv[2] if len(sys.argv) > 2 else "verified")
print(json.dumps({"probe_s": time.perf_counter() - t0, "genes": ev.gene_length,
                  "dropped": {l: m for l, m in ev.probe_log.items() if not m.startswith("verified")}}), flush=True)
ev.prepare()
for pop, gens in ((20, 10),):
    t0 = time.perf_counter()
    res = ga.run_ga(ga.GAConfig(population=pop, generations=gens, rng_seed=0), ev.gene_length, ev)
    el = time.perf_counter() - t0
    ok = sum(1 for r in res.records for i in r.individuals if i.eval_source == "fresh" and i.time_s < 1000)
    print(json.dumps({"ga": app, "pop": pop, "gens": gens, "wall_s": el, "evals": res.evaluations, "valid": ok,
                      "evals_per_s": res.evaluations / el, "gens_per_s": gens / el,
                      "best": ga.genome_str(res.best.genome), "best_ms": res.best.time_s * 1e3,
                      "cpu_ms": ev.measure((0,) * ev.gene_length).seconds * 1e3,
                      "best_loops": [l for l, b in zip(ev.eligible_ids, res.best.genome) if b]}), flush=True)
ev.close()
