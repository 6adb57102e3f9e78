"""The CPU oracle is pinned to the reference's own execution of the program.

Goldens (tests/golden/*.stdout) are the stdout of acctuner's
ExternalEvaluator.run_for_output on the Himeno C-subset text compiled with
"gcc -O2 -w" (oracle/pin_reference.py).  The oracle must print the same
tokens, byte for byte.
"""
import numpy as np
import pytest

from conftest import GOLDEN
from oracle import oracle
from paper_2002_12115_b200.apps import himeno

CASES = [("XXS", 1), ("XXS", 3), ("XS", 1), ("XS", 3), ("S", 2), ("M", 2)]


@pytest.mark.parametrize("name,nn", CASES)
def test_oracle_matches_reference_stdout(name, nn):
    sz = himeno.size(name)
    res = oracle.run_program(sz.I, sz.J, sz.K, nn)
    want = (GOLDEN / f"himeno_{name.lower()}_n{nn}.stdout").read_text().split()
    assert oracle.stdout_lines(res, sz.sample_points()) == want


def test_fp64_gosa_is_sum_of_same_terms():
    sz = himeno.size("XS")
    res = oracle.run_program(sz.I, sz.J, sz.K, 3)
    # fp32 sequential drifts from the fp64 sum but stays close at XS
    assert abs(res["gosa64"] - res["gosa32"]) / res["gosa64"] < 1e-3
    assert res["gosa64"] > 0


def test_threaded_jacobi_identical_field():
    sz = himeno.size("XS")
    a = oracle.empty_fields(sz.I, sz.J, sz.K)
    oracle.initmt(a)
    b = {k: v.copy() for k, v in a.items()}
    g1, _ = oracle.jacobi(a, 3, threads=1)
    g4, _ = oracle.jacobi(b, 3, threads=4)
    assert np.array_equal(a["p"], b["p"]) and np.array_equal(a["wrk2"], b["wrk2"])
    assert abs(g1 - g4) / g1 < 1e-12


def test_program_is_initmt_then_jacobi():
    sz = himeno.size("XXS")
    whole = oracle.run_program(sz.I, sz.J, sz.K, 2)
    f = oracle.empty_fields(sz.I, sz.J, sz.K)
    oracle.initmt(f)
    g64, g32 = oracle.jacobi(f, 2)
    assert np.array_equal(f["p"], whole["fields"]["p"])
    assert g64 == whole["gosa64"] and g32 == whole["gosa32"]


def test_zero_iterations_leave_initial_state():
    sz = himeno.size("XXS")
    res = oracle.run_program(sz.I, sz.J, sz.K, 0)
    p = res["fields"]["p"]
    imax = sz.I - 1
    i = 3
    assert p[i, 1, 1] == np.float32(i * i) / np.float32((imax - 1) * (imax - 1))
    assert res["gosa64"] == 0.0


def test_parallel_first_touch_initmt_is_initmt():
    sz = himeno.custom_size(21, 17, 40)
    a = oracle.empty_fields(sz.I, sz.J, sz.K)
    b = oracle.empty_fields(sz.I, sz.J, sz.K)
    oracle.initmt(a)
    oracle.initmt_parallel(b, 4)
    for name in oracle.FIELDS:
        assert np.array_equal(a[name], b[name]), name


def test_cpu_bench_subprocess_reports_its_procedure():
    """bench.py's two CPU legs share this procedure (fresh process, bound threads)."""
    from oracle import cpu_bench
    r = cpu_bench.run_subprocess("XS", 0.2, 2, min_iters=3)
    assert r["value"] > 0 and r["cores"] == 2 and r["iterations"] >= 3
    assert r["omp"]["OMP_PROC_BIND"] and "first touch" in r["sample"]
