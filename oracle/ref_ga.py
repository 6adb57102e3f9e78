"""The reference's GA fitness path on the host CPU.  REFERENCE ARM / TEST INFRASTRUCTURE.

Reproduces what ``acctuner`` does per fresh genome with its external evaluator
(pkg/src/acctuner/evaluators.py:190-222): write the program text into a temp
dir, compile it with the compile template, run the binary and time the run with
``perf_counter``; ``max_concurrency`` evaluations in flight
(ga.py:222-230).  With a host compiler the OpenACC pragmas are ignored, so
every genome's variant is the all-CPU program; the emitted
pragma lines do not change gcc's work, so the plain program text is compiled.
The GA driving it is paper_2002_12115_b200.ga, bit-exact with acctuner.ga
(tests/test_ga.py).  Used by ``bench.py --impl reference`` only.
"""

from __future__ import annotations

import os
import subprocess
import tempfile
import time
from pathlib import Path
from time import perf_counter

from paper_2002_12115_b200 import ga
from paper_2002_12115_b200.apps import himeno
from paper_2002_12115_b200.evaluator import MeasuredTime

COMPILE = "gcc -O2 -w -mcmodel=medium {src} -o {bin}"
COMPILE_LM = "gcc -O2 -w -mcmodel=medium {src} -o {bin} -lm"   # FT calls exp / sin / cos
RUN = "{bin}"


class ExternalProcedure:
    """acctuner ExternalEvaluator's compile+run procedure on one program text."""

    deterministic = False

    def __init__(self, text: str, file_id: str, timeout_s: float = 180.0,
                 max_concurrency: int = 1, compile_cmd: str = COMPILE):
        self.compile_cmd = compile_cmd
        self.text = text
        self.file_id = file_id
        self.timeout_s = timeout_s
        self.max_concurrency = max_concurrency

    def measure(self, genome) -> MeasuredTime:
        with tempfile.TemporaryDirectory(prefix="acctune-") as tmp:
            src = Path(tmp) / self.file_id
            src.write_text(self.text)
            binary = str(Path(tmp) / "app")
            comp = subprocess.run(self.compile_cmd.format(src=src, bin=binary), shell=True,
                                  capture_output=True, text=True, cwd=tmp)
            if comp.returncode != 0:
                return MeasuredTime.failed("compile failed: " + comp.stderr[-300:])
            t0 = perf_counter()
            try:
                run = subprocess.run(RUN.format(bin=binary), shell=True, capture_output=True,
                                     text=True, cwd=tmp, timeout=self.timeout_s)
            except subprocess.TimeoutExpired:
                return MeasuredTime.timeout()
            elapsed = perf_counter() - t0
            if run.returncode != 0:
                return MeasuredTime.failed("run failed: " + run.stderr[-300:])
            return MeasuredTime.ok(max(elapsed, 1e-9))


def ga_throughput(size_name: str, nn: int, pop: int, gens: int, seed: int,
                  workers: int = 0) -> dict:
    sz = himeno.size(size_name)
    workers = workers or (os.cpu_count() or 1)
    ev = ExternalProcedure(himeno.source_text(sz, nn), himeno.source_file_id(sz),
                           max_concurrency=workers)
    t0 = time.perf_counter()
    res = ga.run_ga(ga.GAConfig(population=pop, generations=gens, rng_seed=seed),
                    himeno.program().gene_length, ev)
    el = time.perf_counter() - t0
    return {"size": size_name, "nn": nn, "population": pop, "generations": gens, "seed": seed,
            "workers": workers, "wall_s": el, "fresh_evals": res.evaluations,
            "evals_per_s": res.evaluations / el, "gens_per_s": gens / el,
            "best_genome": ga.genome_str(res.best.genome), "best_time_s": res.best.time_s,
            "procedure": "acctuner ExternalEvaluator: gcc -O2 compile + run + perf_counter "
                         "per fresh genome (pragmas ignored by gcc)"}


def ft_ga_throughput(cls: str, pop: int, gens: int, seed: int, workers: int = 0) -> dict:
    """The same procedure on the NAS FT restatement (apps/ft.py)."""
    from paper_2002_12115_b200.apps import ft
    c = ft.ft_class(cls)
    workers = workers or (os.cpu_count() or 1)
    ev = ExternalProcedure(ft.source_text(c), ft.source_file_id(c), max_concurrency=workers,
                           compile_cmd=COMPILE_LM)
    t0 = time.perf_counter()
    res = ga.run_ga(ga.GAConfig(population=pop, generations=gens, rng_seed=seed),
                    ft.program(c).gene_length, ev)
    el = time.perf_counter() - t0
    return {"app": f"ft_{c.name.lower()}", "population": pop, "generations": gens, "seed": seed,
            "workers": workers, "wall_s": el, "fresh_evals": res.evaluations,
            "evals_per_s": res.evaluations / el, "gens_per_s": gens / el,
            "best_genome": ga.genome_str(res.best.genome), "best_time_s": res.best.time_s,
            "procedure": "acctuner ExternalEvaluator: gcc -O2 -lm compile + run per fresh genome "
                         "(pragmas ignored by gcc: every genome is the all-CPU program)"}
