import sys, os, random
sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..", "..")))
sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..", "..", "tests")))
from paper_2002_12115_b200 import generic
from paper_2002_12115_b200.apps import ft
from test_generic import _ft_exact_ids
prog = ft.program("S")
exact = _ft_exact_ids(prog)
with generic.GenEvaluator("ft_s", devices=[0], nested_policy="outermost") as ev:
    pats = [tuple(int(l in exact) for l in ev.eligible_ids)]
    rng = random.Random(3)
    for _ in range(3):
        pats.append(tuple(rng.randint(0, 1) for _ in range(ev.gene_length)))
    for g in pats:
        m = ev.measure(g)
        print("pattern", sum(g), "genes on:", m.seconds, m.failure, ft.checksum_error(ev.outputs.get(g, ""), "S"))
