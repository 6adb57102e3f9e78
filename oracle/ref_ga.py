"""The reference's GA fitness path on the host CPU.  REFERENCE ARM / TEST INFRASTRUCTURE.

Reproduces what ``acctuner`` does per fresh genome with its external evaluator
(pkg/src/acctuner/evaluators.py:190-222): write the program text into a temp
dir, compile it with the compile template, run the binary and time the run with
``perf_counter``; ``max_concurrency`` evaluations in flight
(ga.py:222-230).  With a host compiler the OpenACC pragmas are ignored, so
every genome's variant is the all-CPU program; the emitted
pragma lines do not change gcc's work, so the plain program text is compiled.
When the unmodified reference package is available (``baseline/_ref``, installed
by ``__graft_entry__.build()``, or ``/root/reference/pkg/src``) the GA line runs
*the reference itself*: ``acctuner.code_model.analyze_project`` ->
``classify_project`` -> ``ExternalEvaluator(CommandConfig, build_variant)`` exactly
as ``cli.build_evaluator`` builds it (cli.py:108-122), driven by
``acctuner.ga.run_ga``.  Otherwise the restated procedure below, driven by
paper_2002_12115_b200.ga (bit-exact with acctuner.ga, tests/test_ga.py).  Used by
``bench.py --impl reference`` only.
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


ROOT = Path(__file__).resolve().parents[1]
REFERENCE_PATHS = (ROOT / "baseline" / "_ref", Path("/root/reference/pkg/src"))


def reference_package():
    """Import the unmodified acctuner package if one is available (else None)."""
    import sys
    for p in REFERENCE_PATHS:
        if (p / "acctuner" / "ga.py").exists():
            if str(p) not in sys.path:
                sys.path.append(str(p))
            import acctuner.ga  # noqa: F401
            return p
    return None


def reference_ga_throughput(text: str, file_id: str, pop: int, gens: int, seed: int,
                            workers: int, compile_cmd: str) -> dict:
    """The reference's own tune path (cli.py:211-247) minus reports: parse, classify
    with the static probe, ExternalEvaluator over gcc, acctuner.ga.run_ga."""
    from acctuner.classify import StaticRuleProbe, classify_project, eligible_ids
    from acctuner.code_model import analyze_project
    from acctuner.emitter import emit_variant
    from acctuner.evaluators import CommandConfig, ExternalEvaluator
    from acctuner.ga import GAConfig, genome_str, run_ga
    from acctuner.transfer import Planner
    project = analyze_project([(file_id, text)])
    verdicts = classify_project(project, StaticRuleProbe())
    elig = eligible_ids(verdicts)
    planner = Planner(project.loops, project.refs, elig)

    def build_variant(genome):
        return emit_variant(project, genome, verdicts, planner.plan(genome))

    ev = ExternalEvaluator(CommandConfig(compile_cmd, RUN, 180.0, workers), build_variant)
    t0 = time.perf_counter()
    res = run_ga(GAConfig(population=pop, generations=gens, rng_seed=seed), len(elig), ev)
    el = time.perf_counter() - t0
    failed = sum(1 for r in res.records for i in r.individuals if i.eval_source == "penalty")
    return {"wall_s": el, "fresh_evals": res.evaluations,
            "executed_evals": res.evaluations - failed,
            "executed_evals_per_s": (res.evaluations - failed) / el,
            "fresh_evals_per_s": res.evaluations / el, "gens_per_s": gens / el,
            "best_genome": genome_str(res.best.genome), "best_time_s": res.best.time_s,
            "gene_length": len(elig),
            "procedure": "the unmodified reference (acctuner from baseline/_ref): "
                         "analyze_project -> classify_project(StaticRuleProbe) -> "
                         f"ExternalEvaluator('{compile_cmd}', '{RUN}') -> acctuner.ga.run_ga "
                         "(gcc ignores the emitted OpenACC pragmas)"}


def ga_throughput(size_name: str, nn: int, pop: int, gens: int, seed: int,
                  workers: int = 0) -> dict:
    sz = himeno.size(size_name)
    workers = workers or (os.cpu_count() or 1)
    head = {"size": size_name, "nn": nn, "population": pop, "generations": gens, "seed": seed,
            "workers": workers}
    if reference_package() is not None:
        return head | reference_ga_throughput(himeno.source_text(sz, nn),
                                              himeno.source_file_id(sz), pop, gens, seed,
                                              workers, COMPILE)
    ev = ExternalProcedure(himeno.source_text(sz, nn), himeno.source_file_id(sz),
                           max_concurrency=workers)
    t0 = time.perf_counter()
    res = ga.run_ga(ga.GAConfig(population=pop, generations=gens, rng_seed=seed),
                    himeno.program().gene_length, ev)
    el = time.perf_counter() - t0
    return head | {
            "wall_s": el, "fresh_evals": res.evaluations, "executed_evals": res.evaluations,
            "executed_evals_per_s": res.evaluations / el,
            "fresh_evals_per_s": res.evaluations / el, "gens_per_s": gens / el,
            "best_genome": ga.genome_str(res.best.genome), "best_time_s": res.best.time_s,
            "procedure": "acctuner ExternalEvaluator: gcc -O2 compile + run + perf_counter "
                         "per fresh genome (pragmas ignored by gcc)"}


def ft_ga_throughput(cls: str, pop: int, gens: int, seed: int, workers: int = 0) -> dict:
    """The same procedure on the NAS FT restatement (apps/ft.py)."""
    from paper_2002_12115_b200.apps import ft
    c = ft.ft_class(cls)
    workers = workers or (os.cpu_count() or 1)
    head = {"app": f"ft_{c.name.lower()}", "population": pop, "generations": gens,
            "seed": seed, "workers": workers}
    if reference_package() is not None:
        return head | reference_ga_throughput(ft.source_text(c), ft.source_file_id(c), pop,
                                              gens, seed, workers, COMPILE_LM)
    ev = ExternalProcedure(ft.source_text(c), ft.source_file_id(c), max_concurrency=workers,
                           compile_cmd=COMPILE_LM)
    t0 = time.perf_counter()
    res = ga.run_ga(ga.GAConfig(population=pop, generations=gens, rng_seed=seed),
                    ft.program(c).gene_length, ev)
    el = time.perf_counter() - t0
    return head | {
            "wall_s": el, "fresh_evals": res.evaluations, "executed_evals": res.evaluations,
            "executed_evals_per_s": res.evaluations / el,
            "fresh_evals_per_s": res.evaluations / el, "gens_per_s": gens / el,
            "best_genome": ga.genome_str(res.best.genome), "best_time_s": res.best.time_s,
            "procedure": "acctuner ExternalEvaluator: gcc -O2 -lm compile + run per fresh genome "
                         "(pragmas ignored by gcc: every genome is the all-CPU program)"}
