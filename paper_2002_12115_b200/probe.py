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

With ``execute=True`` (a GPU is needed) a table hit is then *run*, which is stronger
than the reference's trial compile: the one-gene pattern that puts only this loop on the
device, under this kind, is executed on a small grid through the real evaluator
(NaN-poisoned device memory, coherence-guarded plan), and the loop is accepted only if p
(bit for bit) and gosa (1e-12 relative) equal the all-CPU program's.  Results are cached
per (loop, kind).

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
    """Accepts (loop, kind) iff the B200 executor implements that loop under that kind
    (and, with ``execute=True``, iff running it reproduces the all-CPU program)."""

    name = "b200"
    max_concurrency = 0

    def __init__(self, program=None, execute: bool = False, size: str = "XS", nn: int = 2,
                 device: int = 0):
        self._program = program or himeno.program()
        model = self._program.model
        self._table = {l.loop_id: (l.parent_loop, _shape(l.shape)) for l in model.loops}
        self.execute = bool(execute)
        self._size, self._nn, self._device = size, int(nn), int(device)
        self._evaluators: dict = {}     # kind value -> (B200Evaluator, all-CPU p, gosa)
        self._cache: dict = {}          # (loop id, kind value) -> ProbeResult

    def _run_probe(self, lid: int, kind_value: str) -> tuple:
        """(accepted, diagnostic): the one-gene pattern of `lid` under `kind_value`
        against the all-CPU program, on the probe's small grid."""
        import numpy as np
        from .errors import BaselineFailure
        from .evaluator import B200Evaluator
        from .kinds import DirectiveKind
        ent = self._evaluators.get(kind_value)
        if ent is None:
            kind = DirectiveKind(kind_value)
            ev = B200Evaluator(self._size, nn=self._nn, devices=[self._device],
                               kinds={l: kind for l in self._program.kinds},
                               poison_device=True)
            base = ev.run((0,) * ev.gene_length)
            ent = (ev, ev.read_field("p", side=0).copy(), float(base.gosa))
            self._evaluators[kind_value] = ent
        ev, p_ref, g_ref = ent
        if lid not in ev.eligible_ids:
            return False, f"loop {lid} is not a gene of the program"
        genome = tuple(int(l == lid) for l in ev.eligible_ids)
        try:
            res = ev.run(genome)
        except BaselineFailure as exc:
            return False, f"execution failed: {exc}"
        p = ev.read_field("p", side=0)
        if not np.array_equal(p, p_ref):
            return False, f"p differs from the all-CPU program ({int((p != p_ref).sum())} points)"
        if abs(float(res.gosa) - g_ref) > 1e-12 * max(abs(g_ref), 1e-300):
            return False, f"gosa {float(res.gosa):.9e} != all-CPU {g_ref:.9e}"
        return True, f"executed on {self._size} nn={self._nn}: p bit-exact, gosa equal"

    def close(self) -> None:
        for ev, _, _ in self._evaluators.values():
            ev.close()
        self._evaluators.clear()

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
        if self.execute:
            key = (lid, kind_value)
            hit = self._cache.get(key)
            if hit is None:
                ok, run_diag = self._run_probe(lid, kind_value)
                hit = ProbeResult(ok, "; ".join(d for d in (diag, run_diag) if d),
                                  (perf_counter() - t0) * 1e3)
                self._cache[key] = hit
            return hit
        return ProbeResult(True, diag, (perf_counter() - t0) * 1e3)
