"""The library's NCCL transport (hp_dd_init / hp_dd_jacobi: halo send/recv, overlapped with
the interior, and the gosa all-reduce) with several ranks on ONE GPU: real NCCL refuses two
ranks on one device, so the library loads a test-only stand-in (tests/nccl_shim.cpp,
HIMENO_NCCL_LIB) that keeps NCCL's stream-ordering semantics, with the ranks as threads of
one process, each driving its own slab context.  The assembled field must equal the
full-grid oracle bit for bit, the all-reduced gosa within 1e-12, on every rank."""
import json
import os
import shutil
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]

SCRIPT = r"""
import json, sys, threading
import numpy as np
sys.path.insert(0, {root!r})
from oracle import oracle
from paper_2002_12115_b200 import dd, native as N
from paper_2002_12115_b200.apps import himeno

ranks, name, nn = {ranks}, {name!r}, {nn}
sz = himeno.size(name)
N.load().hp_set_temporal_blocking({tb})
uid = N.nccl_unique_id()
ctxs = [N.Context(0, sz.I, sz.J, sz.K, slab=dd.slab_range(sz.I, ranks, r)) for r in range(ranks)]
for c in ctxs:
    c.init_device()
out = [None] * ranks
err = []
def run(r):
    try:
        c = ctxs[r]
        c.dd_init(ranks, r, uid)
        c.dd_jacobi(nn)
        c.sync()
        out[r] = (c.read_gosa(1), c.read_field("p", 1)[dd.HALO:-dd.HALO])
    except Exception as exc:   # reported below
        err.append(repr(exc))
ts = [threading.Thread(target=run, args=(r,)) for r in range(ranks)]
for t in ts: t.start()
for t in ts: t.join(300)
if err or any(t.is_alive() for t in ts):
    print(json.dumps({{"ok": False, "err": err or ["timeout"]}})); sys.exit(0)
ref = oracle.run_program(sz.I, sz.J, sz.K, nn)
p = ref["fields"]["p"].copy()
for r in range(ranks):
    b, e = dd.slab_range(sz.I, ranks, r)
    p[b:e] = out[r][1]
same = bool(np.array_equal(p, ref["fields"]["p"]))
g = [o[0] for o in out]
print(json.dumps({{"ok": True, "same": same, "gosa": g, "want": ref["gosa64"]}}))
for c in ctxs:
    c.close()
"""


@pytest.fixture(scope="module")
def shim(tmp_path_factory):
    cuda = Path(os.environ.get("CUDA_HOME", "/usr/local/cuda"))
    gxx = shutil.which("g++")
    if not gxx:
        pytest.skip("g++ not available")
    out = tmp_path_factory.mktemp("shim") / "libnccl_shim.so"
    subprocess.run([gxx, "-O2", "-shared", "-fPIC", "-std=c++17", f"-I{cuda / 'include'}",
                    str(ROOT / "tests" / "nccl_shim.cpp"), f"-L{cuda / 'lib64'}", "-lcudart",
                    "-o", str(out)], check=True)
    return out


@pytest.mark.gpu
@pytest.mark.parametrize("ranks,name,nn,tb,overlap", [
    (2, "XS", 4, 1, 1), (3, "XS", 5, 1, 1), (2, "XS", 3, 0, 0),
    (4, "M", 6, 1, 1), (2, "M", 4, 1, 0), (3, "M", 6, 1, 2),
])
def test_nccl_transport_multi_rank_one_gpu(gpu, shim, ranks, name, nn, tb, overlap):
    # overlap 1: one signalled launch per pass (cuStreamWaitValue32 gates the exchange);
    # 2: two launches (boundary, interior) and an event; 0: exchange after the pass
    env = dict(os.environ, HIMENO_NCCL_LIB=str(shim), HIMENO_DD_OVERLAP=str(min(overlap, 1)),
               HIMENO_DD_SIGNAL="0" if overlap == 2 else "1")
    script = SCRIPT.format(root=str(ROOT), ranks=ranks, name=name, nn=nn, tb=tb)
    proc = subprocess.run([sys.executable, "-c", script], env=env, capture_output=True,
                          text=True, timeout=600)
    assert proc.returncode == 0, proc.stderr[-2000:]
    res = json.loads(proc.stdout.strip().splitlines()[-1])
    assert res["ok"], res
    assert res["same"]
    for g in res["gosa"]:       # every rank holds the all-reduced gosa
        assert abs(g - res["want"]) <= 1e-12 * res["want"]
