"""ctypes wrapper of the CPU oracle (oracle/himeno_oracle.c).  TEST INFRASTRUCTURE ONLY.

Importable by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs -- never by the product package.
"""

from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "_build" / "libhimeno_oracle.so"
FIELDS = ("p", "bnd", "wrk1", "wrk2", "a0", "a1", "a2", "a3",
          "b0", "b1", "b2", "c0", "c1", "c2")

_lib = None


def build() -> Path:
    src = HERE / "himeno_oracle.c"
    if not LIB.exists() or LIB.stat().st_mtime < src.stat().st_mtime:
        LIB.parent.mkdir(exist_ok=True)
        subprocess.run(["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-fopenmp",
                        "-shared", "-o", str(LIB), str(src)], check=True)
    return LIB


def lib():
    global _lib
    if _lib is None:
        build()
        l = C.CDLL(str(LIB))
        P = C.POINTER(C.c_void_p)
        l.oracle_run.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, P,
                                 C.POINTER(C.c_double), C.POINTER(C.c_float)]
        l.oracle_initmt.argtypes = [C.c_int, C.c_int, C.c_int, P]
        l.oracle_jacobi.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, P, C.c_int,
                                    C.POINTER(C.c_double), C.POINTER(C.c_float)]
        l.oracle_initmt_par.argtypes = [C.c_int, C.c_int, C.c_int, P, C.c_int]
        l.oracle_max_threads.restype = C.c_int
        _lib = l
    return _lib


def empty_fields(I: int, J: int, K: int) -> dict:
    """The program's static arrays: zero-initialised."""
    return {name: np.zeros((I, J, K), dtype=np.float32) for name in FIELDS}


def _ptrs(fields: dict):
    arr = (C.c_void_p * len(FIELDS))()
    for idx, name in enumerate(FIELDS):
        a = fields[name]
        assert a.dtype == np.float32 and a.flags.c_contiguous
        arr[idx] = a.ctypes.data
    return arr


def run_program(I: int, J: int, K: int, nn: int) -> dict:
    """initmt + jacobi(nn) sequentially; returns fields + gosa (fp64 and literal fp32)."""
    f = empty_fields(I, J, K)
    g64, g32 = C.c_double(), C.c_float()
    rc = lib().oracle_run(I, J, K, nn, _ptrs(f), C.byref(g64), C.byref(g32))
    if rc != 0:
        raise ValueError("oracle_run: bad arguments")
    return {"fields": f, "gosa64": g64.value, "gosa32": g32.value}


def initmt(fields: dict) -> None:
    I, J, K = fields["p"].shape
    if lib().oracle_initmt(I, J, K, _ptrs(fields)) != 0:
        raise ValueError("oracle_initmt: bad arguments")


def initmt_parallel(fields: dict, threads: int) -> None:
    """initmt with NUMA-friendly first touch (planes by the threads that compute them)."""
    I, J, K = fields["p"].shape
    if lib().oracle_initmt_par(I, J, K, _ptrs(fields), threads) != 0:
        raise ValueError("oracle_initmt_par: bad arguments")


def jacobi(fields: dict, nn: int, threads: int = 1) -> tuple:
    """jacobi(nn) in place; returns (gosa64, gosa32)."""
    I, J, K = fields["p"].shape
    g64, g32 = C.c_double(), C.c_float()
    if lib().oracle_jacobi(I, J, K, nn, _ptrs(fields), threads, C.byref(g64), C.byref(g32)) != 0:
        raise ValueError("oracle_jacobi: bad arguments")
    return g64.value, g32.value


def max_threads() -> int:
    return int(lib().oracle_max_threads())


def stdout_lines(result: dict, samples) -> list:
    """What the program prints: fp32 gosa then the p samples, "%.9e"."""
    p = result["fields"]["p"]
    return [f"{result['gosa32']:.9e}"] + [f"{float(p[i, j, k]):.9e}" for i, j, k in samples]
