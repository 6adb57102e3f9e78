import sys, os, json, time
sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..", "..")))
sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..", "..", "tests")))
from paper_2002_12115_b200 import generic
from paper_2002_12115_b200.apps import ft
from test_generic import _ft_exact_ids
for app, cls in (("ft_w", "W"), ("ft_a", "A")):
    prog = ft.program(cls)
    exact = _ft_exact_ids(prog)
    bulk = [l for l in exact if prog.model.loops.get(l).index_var in ("k", "j") and prog.model.loops.get(l).parent_loop is None or l in (3, 4)]
    with generic.GenEvaluator(app, devices=[0]) as ev:
        for name, on in (("cpu", []), ("exact", exact), ("bulk", bulk)):
            g = tuple(int(l in on) for l in ev.eligible_ids)
            ts = [ev.measure(g).seconds for _ in range(2)]
            st = ev.stats[g]
            print(json.dumps({"app": app, "pattern": name, "loops": on, "ms": [round(t * 1e3, 1) for t in ts],
                              "launches": st["n_launch"], "h2d_MB": st["h2d_bytes"] / 1e6,
                              "d2h_MB": st["d2h_bytes"] / 1e6, "err": ft.checksum_error(ev.outputs[g], cls)}), flush=True)
