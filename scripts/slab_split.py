"""L in 8 slabs (virtual ranks on one GPU, in-process group): jacobi(40) wall time with the
halo exchange after each whole pass vs overlapped (boundary launch + interior launch), and
with the exchange kernel for whole passes.  On one GPU the 8 slabs share the device, so this
measures the split's extra work, not the overlap's benefit."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2002_12115_b200 import dd  # noqa: E402

for ranks in (8, 4):
    with dd.GroupJacobi("L", [0] * ranks) as g:
        for rep in range(2):
            for conf in (("1", "0", "1"), ("1", "0", "0"), ("0", "0", "1"), ("0", "1", "1")):
                os.environ["HIMENO_DD_OVERLAP"], os.environ["HIMENO_TX"], os.environ["HIMENO_DD_SIGNAL"] = conf
                g.jacobi(8)
                t0 = time.perf_counter()
                g.jacobi(40)
                el = time.perf_counter() - t0
                print(f"L/{ranks} overlap={conf[0]} tx={conf[1]} signal={conf[2]}: {el * 1e3 / 20:.3f} ms per two-step pass "
                      f"(all {ranks} slabs on one GPU)", flush=True)
