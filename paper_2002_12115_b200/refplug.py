"""Reference-side binding: the B200 evaluator selected from acctuner's own pipeline.

``build_b200_evaluator(cfg, project, verdicts)`` is what the reference's
``build_evaluator`` (``acctuner/cli.py:108-122``) returns for
``evaluator.type == "b200"``.  It returns an instance of an
``acctuner.evaluators.ExternalEvaluator`` subclass, so every reference code path
that dispatches on the plugin type runs unchanged:

* ``run_ga`` / ``_evaluate_generation`` call ``measure(genome)`` on
  ``max_concurrency`` pool threads (``ga.py:214-245``);
* ``measure_baseline`` measures the all-zero genome (``cli.py:200-208``);
* ``run_pipeline``'s verification branch (``cli.py:263-271``,
  ``isinstance(evaluator, ExternalEvaluator)``) calls ``run_for_output(texts)``
  with the original program texts and with the emitted best variant.

What replaces compile+run is ``B200Evaluator`` (evaluator.py): the genome's
``Planner.plan`` is lowered to a schedule and executed by libhimeno_b200.so.
``run_for_output`` receives *texts*, not a genome (``evaluators.py:183-188``);
the genome is recovered by matching the texts against the original program and
the reference's own ``emit_variant`` of the genomes this evaluator has seen.

This module imports ``acctuner`` lazily: the product path (B200Evaluator) never
depends on the reference package.
"""

from __future__ import annotations

import re
import threading

from .errors import BaselineFailure, ConfigError, EvaluatorUnavailable
from .evaluator import B200Evaluator


def _program_nn(project) -> int:
    """jacobi's iteration count as the program text passes it (``gosa = jacobi(N);``)."""
    for unit in project.units:
        m = re.search(r"\bjacobi\s*\(\s*(\d+)\s*\)", unit.original_text)
        if m:
            return int(m.group(1))
    raise ConfigError("cannot find the jacobi(N) call in the program text; set evaluator.nn")


def reference_evaluator_class():
    """The ExternalEvaluator subclass (created on first use; needs acctuner)."""
    global _CLS
    if _CLS is not None:
        return _CLS
    from acctuner import errors as ref_errors
    from acctuner.emitter import emit_variant
    from acctuner.evaluators import ExternalEvaluator
    from acctuner.evaluators import MeasuredTime as RefMeasuredTime
    from acctuner.transfer import Planner as RefPlanner

    class B200ExternalEvaluator(ExternalEvaluator):
        """ExternalEvaluator whose compile+run is one hp_run on a B200."""

        deterministic = False

        def __init__(self, b200: B200Evaluator, project, verdicts, elig):
            # no CommandConfig: the library replaces the compile/run templates
            self.config = None
            self.b200 = b200
            self.project = project
            self.verdicts = verdicts
            self.planner = RefPlanner(project.loops, project.refs, elig)
            self.max_concurrency = b200.max_concurrency
            self._seen: list = []
            self._seen_lock = threading.Lock()

        def build_variant(self, genome):   # the reference's build_variant (cli.py:119-120)
            return emit_variant(self.project, genome, self.verdicts, self.planner.plan(genome))

        def measure(self, genome):
            genome = tuple(int(b) for b in genome)
            with self._seen_lock:
                self._seen.append(genome)
            try:
                m = self.b200.measure(genome)
            except EvaluatorUnavailable as exc:   # -> the reference CLI's exit code 2
                raise ref_errors.EvaluatorUnavailable(str(exc)) from exc
            if m.failure is not None:
                return RefMeasuredTime.failed(m.failure)
            if m.timed_out:
                return RefMeasuredTime.timeout()
            return RefMeasuredTime.ok(m.seconds)

        def genome_of(self, texts: dict) -> tuple:
            n = self.b200.gene_length
            originals = {u.file_id: u.original_text for u in self.project.units}
            if dict(texts) == originals:
                return (0,) * n
            with self._seen_lock:
                seen = list(dict.fromkeys(reversed(self._seen)))
            for g in seen:
                if self.build_variant(g).texts == dict(texts):
                    return g
            raise ConfigError("run_for_output: texts are neither the original program nor "
                              "a variant of a genome this evaluator measured")

        def run_for_output(self, texts: dict) -> str:
            # verification path: main's stdout under the variant's pattern, with the
            # literal fp32 gosa (evaluator.B200Evaluator.run_for_output)
            try:
                return self.b200.run_for_output(self.genome_of(texts))
            except BaselineFailure as exc:
                # a variant that does not run (evaluators.py:186-187); the reference's
                # exception type, so run_pipeline / main handle it as their own
                raise ref_errors.BaselineFailure(str(exc)) from exc

        def close(self) -> None:
            self.b200.close()

    _CLS = B200ExternalEvaluator
    return _CLS


_CLS = None


def build_b200_evaluator(cfg, project, verdicts):
    """``build_evaluator`` for ``evaluator.type == "b200"`` (cli.py:108-122).

    Keys of ``cfg.evaluator``: ``size`` (default: inferred from p's extents),
    ``nn`` (default: the program's ``jacobi(N)``), ``devices`` (list or "all"),
    ``workers_per_device``, ``transfer_mode``, ``nested_policy``, ``timeout_s``.
    """
    from acctuner.classify import eligible_ids
    e = dict(getattr(cfg, "evaluator", None) or {})
    nn = int(e["nn"]) if "nn" in e else _program_nn(project)
    elig = eligible_ids(verdicts)
    b200 = B200Evaluator.from_project(
        project, verdicts, size=e.get("size"), nn=nn, devices=e.get("devices", [0]),
        workers_per_device=int(e.get("workers_per_device", 1)),
        transfer_mode=e.get("transfer_mode", "batched"),
        nested_policy=e.get("nested_policy", "reject"),
        timeout_s=float(e.get("timeout_s", 180.0)))
    return reference_evaluator_class()(b200, project, verdicts, elig)
