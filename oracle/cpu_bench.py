"""CPU baseline of the Himeno Jacobi: the oracle's OpenMP jacobi.  TEST INFRASTRUCTURE ONLY.

Used by bench.py for BOTH CPU legs -- the ``cpu_baseline`` object of the B200 arm
and the ``--impl reference`` arm -- so the two report the same procedure:

* a fresh process (``python -m oracle.cpu_bench``; no CUDA context, no torch
  thread pool competing for the cores), launched with ``OMP_PROC_BIND=spread``
  and ``OMP_PLACES=cores`` unless the caller set them;
* the fields first-touched in parallel by the threads that compute their
  planes (``oracle_initmt_par``: same static schedule over i as the jacobi);
* one untimed iteration, then whole iterations until ``--seconds`` have passed
  (at least ``--min-iters``), each timed; the value is flops / total time.

Prints one JSON object.
"""

from __future__ import annotations

import argparse
import json
import os
import platform
import subprocess
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
FLOP_PER_POINT = 34


def host_threads() -> int:
    try:
        return max(1, len(os.sched_getaffinity(0)))
    except (AttributeError, OSError):
        return max(1, os.cpu_count() or 1)


def numa_nodes() -> int:
    try:
        return len([d for d in os.listdir("/sys/devices/system/node") if d.startswith("node")])
    except OSError:
        return 1


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor() or "unknown"


def measure(size_name: str, seconds: float, threads: int, min_iters: int = 1,
            max_iters: int = 1000, warmup: int = 1) -> dict:
    sys.path.insert(0, str(ROOT))
    from oracle import oracle
    from paper_2002_12115_b200.apps import himeno
    sz = himeno.size(size_name)
    f = oracle.empty_fields(sz.I, sz.J, sz.K)
    oracle.initmt_parallel(f, threads)
    for _ in range(max(1, warmup)):
        oracle.jacobi(f, 1, threads=threads)      # untimed
    times = []
    t_all = time.perf_counter()
    while True:
        t0 = time.perf_counter()
        oracle.jacobi(f, 1, threads=threads)
        times.append(time.perf_counter() - t0)
        if (len(times) >= min_iters and time.perf_counter() - t_all >= seconds) or \
                len(times) >= max_iters:
            break
    total = sum(times)
    flops = FLOP_PER_POINT * sz.interior_points
    return {"value": flops * len(times) / total / 1e9, "unit": "GFLOP/s", "cores": threads,
            "kind": "port", "iterations": len(times),
            "best_iter_gflops": flops / min(times) / 1e9,
            "median_iter_s": sorted(times)[len(times) // 2],
            "sample": f"oracle jacobi (C restatement of the program the reference compiles, "
                      f"gcc -O2 -fopenmp) on Himeno {sz.name} ({sz.I}x{sz.J}x{sz.K}): "
                      f"{len(times)} timed iteration(s), {total:.2f} s, {threads} OpenMP "
                      f"threads, parallel first touch, fresh process",
            "omp": {"OMP_PROC_BIND": os.environ.get("OMP_PROC_BIND"),
                    "OMP_PLACES": os.environ.get("OMP_PLACES")},
            "numa_nodes": numa_nodes(), "cpu": cpu_model()}


def run_subprocess(size_name: str, seconds: float, threads: int, min_iters: int = 1,
                   warmup: int = 1, timeout: float = 600) -> dict:
    """measure() in a fresh interpreter (the bench process holds CUDA contexts and
    torch's own OpenMP pool)."""
    env = dict(os.environ)
    env.setdefault("OMP_PROC_BIND", "spread")
    env.setdefault("OMP_PLACES", "cores")
    env["OMP_NUM_THREADS"] = str(threads)
    out = subprocess.run([sys.executable, "-m", "oracle.cpu_bench", "--size", size_name,
                          "--seconds", str(seconds), "--threads", str(threads),
                          "--min-iters", str(min_iters), "--warmup", str(warmup)],
                         cwd=str(ROOT), env=env, capture_output=True, text=True, timeout=timeout,
                         check=True)
    return json.loads(out.stdout.strip().splitlines()[-1])


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(description=__doc__.splitlines()[0])
    ap.add_argument("--size", default="L")
    ap.add_argument("--seconds", type=float, default=10.0)
    ap.add_argument("--threads", type=int, default=0)
    ap.add_argument("--min-iters", type=int, default=1)
    ap.add_argument("--warmup", type=int, default=1)
    a = ap.parse_args(argv)
    print(json.dumps(measure(a.size, a.seconds, a.threads or host_threads(), a.min_iters,
                             warmup=a.warmup)))
    return 0


if __name__ == "__main__":
    sys.exit(main())
