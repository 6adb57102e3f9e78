import sys, os, json, time
sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..", "..")))
from paper_2002_12115_b200 import generic, ga
from paper_2002_12115_b200.apps import ft
EXACT = [0, 3, 4, 10, 13, 16, 19, 22, 25, 28, 31, 34, 37, 40, 43, 45, 49, 53, 56, 59, 62, 65, 68, 71, 74, 77, 80, 83, 86, 88, 91]
for app in ("ft_s", "ft_w"):
    with generic.GenEvaluator(app, devices=[0]) as ev:
        if app == "ft_w": continue
        if False: pass
        ev.prepare()
        for name, on in [("cpu", []), ("exact", EXACT), ("bulk", [0, 3, 4, 45, 49, 88, 91]),
                         ("ffts", [10, 13, 16, 19, 22, 25, 28, 31, 34, 37, 40, 43, 53, 56, 59, 62, 65, 68, 71, 74, 77, 80, 83, 86])]:
            g = tuple(int(l in on) for l in ev.eligible_ids)
            ts = []
            for _ in range(3):
                m = ev.measure(g); ts.append(m.seconds)
            st = ev.stats[g]
            print(json.dumps({"app": app, "pattern": name, "ms": [round(t*1e3, 2) if t else None for t in ts],
                              "launches": st["n_launch"], "h2d_MB": st["h2d_bytes"]/1e6, "d2h_MB": st["d2h_bytes"]/1e6,
                              "err": ft.checksum_error(ev.outputs[g], app[-1].upper())}), flush=True)
        for lid in ev.eligible_ids:
            g = tuple(int(l == lid) for l in ev.eligible_ids)
            m = ev.measure(g)
            print(json.dumps({"app": app, "single": lid, "note": ev.lib.loop_notes[lid], "ms": m.seconds and round(m.seconds*1e3, 2),
                              "fail": m.failure, "err": ft.checksum_error(ev.outputs.get(g, ""), app[-1].upper())}), flush=True)
with generic.GenEvaluator("ft_s", devices=[0], workers_per_device=4, verify_each=True) as ev:
    ev.prepare()
    t0 = time.perf_counter()
    res = ga.run_ga(ga.GAConfig(population=20, generations=10, rng_seed=0), ev.gene_length, ev)
    el = time.perf_counter() - t0
    print(json.dumps({"ga": "ft_s", "wall_s": el, "evals": res.evaluations, "evals_per_s": res.evaluations/el,
                      "best": ga.genome_str(res.best.genome), "best_ms": res.best.time_s*1e3}))
