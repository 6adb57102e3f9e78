"""Golden values of the bench workload (Himeno L, jacobi(100)) from the CPU oracle.

Writes tests/golden/himeno_l_n100.json: the fp64 gosa after 100 iterations, a
SHA-256 of the final p field and main's p samples.  bench.py checks the gosa of
its post-warm-up step against this value (no oracle run on the GPU box), and
tests/test_gpu_parity.py checks the device field against the hash.

    PYTHONPATH=. python scripts/gen_golden_l100.py
"""
import hashlib
import json
import time
from pathlib import Path

from oracle import oracle
from paper_2002_12115_b200.apps import himeno

ROOT = Path(__file__).resolve().parents[1]


def main():
    sz = himeno.size("L")
    f = oracle.empty_fields(sz.I, sz.J, sz.K)
    oracle.initmt(f)
    t0 = time.time()
    g64, _ = oracle.jacobi(f, 100, threads=oracle.max_threads())
    p = f["p"]
    doc = {"grid": [sz.I, sz.J, sz.K], "nn": 100, "gosa64": g64,
           "p_sha256": hashlib.sha256(p.tobytes()).hexdigest(),
           "p_samples": [[i, j, k, float(p[i, j, k])] for i, j, k in sz.sample_points()],
           "oracle_seconds": round(time.time() - t0, 1)}
    (ROOT / "tests" / "golden" / "himeno_l_n100.json").write_text(json.dumps(doc, indent=1) + "\n")
    print(doc)


if __name__ == "__main__":
    main()
