"""B200 eligibility probe: the analogue of the reference's compile probe.

The reference decides per (loop, directive kind) whether GPU processing is possible by
trial-compiling a one-pragma variant (``CommandProbe``, acctuner/classify.py:234-274) or
by static dependence rules (``StaticRuleProbe``, 200-231), and ``classify_loop``
(281-296) takes the first accepted kind in priority order.  On the B200 path the
question is whether libhimeno_b200.so has a kernel variant for the loop under that
kind -- answered instantly from the executor's loop table (csrc/executor.cpp) instead
of a compiler run:

* every loop of the Himeno program (ids 0-12, matched by id, parent and shape) has a
  variant for each kind: ``kernels`` collapses the tight nest below the loop,
  ``parallel loop`` runs one gang per iteration, ``parallel loop vector`` one CTA;
* loop 6 (the time loop) is accepted as the device-resident *sequential* time loop
   -- the static probe accepts it as a parallel loop although
  it carries p/wrk2 between iterations; the diagnostic records the semantics;
* any other loop is rejected ("no B200 kernel variant"), so a program the library does
  not implement classifies to zero genes instead of failing at run time.

The interface is duck-typed like the reference probes (``name``, ``max_concurrency``,
``probe(loop, kind, project) -> ProbeResult``) so ``classify_loop`` runs unchanged.
"""

from __future__ import annotations

from dataclasses import dataclass
from time import perf_counter

from .apps import himeno


@dataclass(frozen=True)
class ProbeResult:
    accepted: bool
    diagnostic: str = ""
    elapsed_ms: float = 0.0


def _shape(value) -> str:
    return getattr(value, "value", value)


class B200Probe:
    """Accepts (loop, kind) iff the B200 executor implements that loop under that kind."""

    name = "b200"
    max_concurrency = 0

    def __init__(self, program=None):
        model = (program or himeno.program()).model
        self._table = {l.loop_id: (l.parent_loop, _shape(l.shape)) for l in model.loops}

    def probe(self, loop, kind, project=None) -> ProbeResult:
        t0 = perf_counter()
        lid = loop.loop_id
        known = self._table.get(lid)
        if known is None or known != (loop.parent_loop, _shape(loop.shape)):
            return ProbeResult(False, f"no B200 kernel variant for loop {lid}",
                               (perf_counter() - t0) * 1e3)
        kind_value = getattr(kind, "value", kind)
        if kind_value not in ("kernels", "parallel loop", "parallel loop vector"):
            return ProbeResult(False, f"unknown directive kind {kind_value!r}",
                               (perf_counter() - t0) * 1e3)
        diag = ""
        if lid == 6:
            diag = "device-resident sequential time loop (iterations carry p/wrk2)"
        return ProbeResult(True, diag, (perf_counter() - t0) * 1e3)
