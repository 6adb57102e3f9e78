"""Small workload exercising every kernel family, for compute-sanitizer runs."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2002_12115_b200 import native as N  # noqa: E402
from paper_2002_12115_b200.apps import himeno  # noqa: E402
from paper_2002_12115_b200.evaluator import B200Evaluator  # noqa: E402
from paper_2002_12115_b200.kinds import DirectiveKind  # noqa: E402

lib = N.load()
sz = himeno.custom_size(20, 29, 300)
for tb in (0, 1):
    lib.hp_set_temporal_blocking(tb)
    with N.Context(0, sz.I, sz.J, sz.K) as c:
        c.init_device()
        c.jacobi_device(3, 1)
        c.jacobi_device(2, 0)
        print("device jacobi tb", tb, c.read_gosa(1))
lib.hp_set_temporal_blocking(1)
with B200Evaluator("XXS", nn=2) as ev:
    for g in ("0000000100100", "0010010010010", "0100100100100", "1001001000000",
              "0000001000000", "0000000000001"):
        print(g, ev.measure(tuple(int(x) for x in g)))
prog = himeno.program()
with B200Evaluator("XXS", nn=2, kinds={l: DirectiveKind.PARALLEL_LOOP_VECTOR for l in prog.kinds}) as ev:
    print("plv", ev.measure((0, 0, 0, 0, 0, 0, 0, 1, 0, 0, 1, 0, 0)))
from paper_2002_12115_b200 import dd  # noqa: E402
with dd.GroupJacobi("XS", [0, 0, 0]) as g:
    print("group", g.jacobi(2))
# round 2: the flow launch (3 two-step passes in one launch), the overlapped halo
# exchange (boundary launch + interior launch + comm-stream copies), and -- when
# SANITIZE_TX=1 -- the tile-exchange kernel
import os  # noqa: E402
os.environ["HIMENO_TB2_FLOW"] = "1"
os.environ["HIMENO_FLOW_CHUNK"] = "8"
with N.Context(0, sz.I, sz.J, sz.K) as c:
    c.init_device()
    c.jacobi_device(6, 1)
    print("flow", N.last_two_step_kernel(), c.read_gosa(1))
del os.environ["HIMENO_TB2_FLOW"], os.environ["HIMENO_FLOW_CHUNK"]
os.environ["HIMENO_DD_OVERLAP"] = "1"
with dd.GroupJacobi("XS", [0, 0, 0]) as g:
    print("group overlapped", g.jacobi(4))
# the two-step variants the small grid does not pick by default (old producer order,
# per-warp stash), and the double-buffered host upload of hp_jacobi_host (serial and two
# contexts in flight)
import numpy as np  # noqa: E402
for env in ({"HIMENO_TB2_ORD": "0"}, {"HIMENO_TB2_XS": "0"}):
    os.environ.update(env)
    with N.Context(0, sz.I, sz.J, sz.K) as c:
        c.init_device()
        c.jacobi_device(3, 1)
        print("variant", env, c.read_gosa(1))
    for k in env:
        del os.environ[k]
with N.Context(0, sz.I, sz.J, sz.K) as a, N.Context(0, sz.I, sz.J, sz.K) as b:
    a.init_device()
    host = {f: a.read_field(f, 1) for f in N.FIELDS}
    outs = [np.empty_like(host["p"]), np.empty_like(host["p"])]
    print("host serial", a.jacobi_host(host, 3, 1, outs[0]))
    a.jacobi_host_async(host, 3, 1, outs[0])
    b.jacobi_host_async(host, 3, 1, outs[1])
    print("host async", a.sync(), b.sync())
if os.environ.get("SANITIZE_TX") == "1":
    os.environ["HIMENO_TX"] = "2"
    with N.Context(0, sz.I, sz.J, sz.K) as c:
        c.init_device()
        c.jacobi_device(4, 1)
        print("tx", N.last_two_step_kernel(), c.read_gosa(1), c.tx_status())
