"""B200 fitness evaluator: the drop-in replacement of the reference's ExternalEvaluator.

Plugin contract (acctuner/ga.py:222-230, evaluators.py:108-128, 168-188):

* ``measure(genome) -> MeasuredTime`` -- one program execution under the
  gene pattern, timed by host wall clock like ``_compile_and_run``
  (evaluators.py:207-214); pattern failures are *returned* as
  ``MeasuredTime.failed`` (penalty, GA continues), timeouts as
  ``MeasuredTime.timeout``; environment problems *raise*
  ``EvaluatorUnavailable`` (``NativeUnavailable`` / ``DeviceError``).
* ``max_concurrency`` -- number of worker slots (B200s x ``workers_per_device``):
  ``run_ga`` measures up to that many fresh genomes at once (population
  sharding with no collectives).  Each call leases a slot,
  which owns its own device context.
* ``deterministic = False`` -- times are measured.

What replaces compile+run: ``Planner.plan(genome)`` (plan.py, same plan as the
reference) is lowered to native events (lower.py) and executed by
libhimeno_b200.so (csrc/executor.cpp).  Plans/schedules are cached per
genome.  The program's stdout (gosa and the p samples main prints) is
available via ``run_for_output`` for the reference's numeric verification
(cli.py:155-186).
"""

from __future__ import annotations

import queue
import threading
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass
from typing import Optional

from . import native as N
from .apps import himeno
from .errors import ConfigError, EvaluatorUnavailable, BaselineFailure
from .lower import NESTED_POLICIES, lower
from .plan import Planner


@dataclass(frozen=True)
class MeasuredTime:
    """ok(seconds > 0) | timeout() | failed(diag)  (evaluators.py:28-46)."""
    seconds: Optional[float] = None
    timed_out: bool = False
    failure: Optional[str] = None

    @classmethod
    def ok(cls, seconds: float) -> "MeasuredTime":
        if seconds <= 0:
            raise ValueError("measured seconds must be positive")
        return cls(seconds=seconds)

    @classmethod
    def timeout(cls) -> "MeasuredTime":
        return cls(timed_out=True)

    @classmethod
    def failed(cls, diagnostic: str) -> "MeasuredTime":
        return cls(failure=diagnostic or "unspecified failure")


TRANSFER_MODES = ("batched", "per-loop")
# genes = 0 run the library's host loops: "tuned" (g++ -O3 -march=x86-64-v3, the
# program as a tuned application) or "reference" (the program's literal loops built
# like the reference's compile template, gcc -O2: host-heavy patterns cost what the
# reference's binary makes them cost).  Same values either way.
HOST_BUILDS = ("tuned", "reference")


def _size_from_refs(refs):
    ext = refs.vars["p"].extents if "p" in refs.vars else None
    if not ext or len(ext) != 3:
        raise ConfigError("cannot infer the Himeno grid: variable p has no [I][J][K] extent")
    return himeno.custom_size(*ext, name=f"{ext[0]}x{ext[1]}x{ext[2]}")


class B200Evaluator:
    """Evaluate Himeno offload genomes on one or more B200s."""

    deterministic = False

    def __init__(self, size="M", nn: int = 3, devices=None, *, loops=None, refs=None,
                 eligible_ids=None, kinds=None, transfer_mode: str = "batched",
                 nested_policy: str = "reject", coherence_guard: bool = True,
                 fused_time_loop: bool = True, fresh_process: bool = True,
                 poison_device: bool = False, timeout_s: float = 180.0,
                 workers_per_device: int = 1, host_build: str = "tuned"):
        if transfer_mode not in TRANSFER_MODES:
            raise ConfigError(f"transfer_mode must be one of {TRANSFER_MODES}")
        if nested_policy not in NESTED_POLICIES:
            raise ConfigError(f"nested_policy must be one of {NESTED_POLICIES}")
        if nn < 1:
            raise ConfigError("nn must be >= 1")
        if host_build not in HOST_BUILDS:
            raise ConfigError(f"host_build must be one of {HOST_BUILDS}")
        self.host_build = host_build
        prog = himeno.program()
        self.loops = loops if loops is not None else prog.model.loops
        self.refs = refs if refs is not None else prog.model.refs
        self.eligible_ids = list(eligible_ids if eligible_ids is not None else prog.eligible)
        self.kinds = dict(kinds if kinds is not None else prog.kinds)
        self.size = himeno.size(size) if size is not None else _size_from_refs(self.refs)
        self.nn = int(nn)
        self.transfer_mode = transfer_mode
        self.nested_policy = nested_policy
        self.timeout_s = float(timeout_s)
        self.flags = ((N.FLAG_COHERENCE_GUARD if coherence_guard else 0)
                      | (N.FLAG_FUSED_TIME_LOOP if fused_time_loop else 0)
                      | (N.FLAG_FRESH_PROCESS if fresh_process else 0)
                      | (N.FLAG_POISON_DEVICE if poison_device else 0)
                      | (N.FLAG_HOST_REFERENCE if host_build == "reference" else 0))
        N.load()   # fail loudly now: no CPU fallback exists
        if devices is None:
            devices = [0]
        elif devices == "all":
            devices = list(range(N.device_count()))
        # one worker slot per entry; a device may appear several times (several
        # concurrent evaluations on one GPU, each with its own context)
        self.devices = list(devices) * max(1, int(workers_per_device))
        if not self.devices:
            raise EvaluatorUnavailable("no CUDA devices to evaluate on")
        self.max_concurrency = len(self.devices)
        self.planner = Planner(self.loops, self.refs, self.eligible_ids)
        self._contexts: dict = {}
        self._ctx_lock = threading.Lock()
        self._free: "queue.Queue[int]" = queue.Queue()
        for slot in range(len(self.devices)):
            self._free.put(slot)
        self._lowered: dict = {}
        self._low_lock = threading.Lock()
        self.stats: dict = {}          # genome -> native result stats of its last run
        self._last_slot = 0
        self._count_lock = threading.Lock()   # measure() runs on run_ga's pool threads
        self.evaluations = 0

    # -- construction from the reference pipeline objects ----------------------
    @classmethod
    def from_project(cls, project, verdicts, size=None, **kw) -> "B200Evaluator":
        """Build from a reference ProjectModel + classify verdicts (cli.py:108-122)."""
        from .kinds import eligible_ids as _elig, kind_map as _kmap
        return cls(size=size, loops=project.loops, refs=project.refs,
                   eligible_ids=_elig(verdicts), kinds=_kmap(verdicts), **kw)

    # -- plan / lowering -------------------------------------------------------------
    @property
    def gene_length(self) -> int:
        return len(self.eligible_ids)

    def plan(self, genome):
        genome = tuple(int(b) for b in genome)
        if self.transfer_mode == "batched":
            return self.planner.plan(genome)
        return self.planner.plan_transfers(genome)

    def lowered(self, genome):
        genome = tuple(int(b) for b in genome)
        with self._low_lock:
            low = self._lowered.get(genome)
        if low is None:
            self.planner.gene_map(genome)   # length check -> GenomeLengthMismatch
            plan = self.plan(genome)
            low = lower(genome, self.eligible_ids, self.kinds, self.loops, self.refs, plan,
                        self.nn, self.flags, self.timeout_s, self.nested_policy)
            with self._low_lock:
                self._lowered[genome] = low
        return low

    # -- device contexts ---------------------------------------------------------------
    def _context(self, slot: int) -> N.Context:
        with self._ctx_lock:
            ctx = self._contexts.get(slot)
            if ctx is None:
                sz = self.size
                ctx = N.Context(self.devices[slot], sz.I, sz.J, sz.K)
                ctx.set_samples(sz.sample_points())
                self._contexts[slot] = ctx
            return ctx

    def prepare(self) -> None:
        """Create every worker slot's device context now (concurrently), instead of
        lazily at the slot's first evaluation."""
        missing = [s for s in range(len(self.devices)) if s not in self._contexts]
        if not missing:
            return
        with ThreadPoolExecutor(max_workers=len(missing)) as pool:
            list(pool.map(self._context, missing))

    def _execute(self, genome, extra_flags: int = 0):
        """Run once in a leased worker slot; returns (lowered, result, slot)."""
        low = self.lowered(genome)
        if low.failure is not None:
            return low, None, None
        sched = low.schedule
        if extra_flags:
            sched = N.Schedule.from_buffer_copy(low.schedule)   # events stay owned by `low`
            sched.flags |= int(extra_flags)
        slot = self._free.get()
        try:
            res = self._context(slot).run(sched)
        finally:
            self._free.put(slot)
        with self._count_lock:
            self._last_slot = slot
        return low, res, slot

    # -- plugin API ----------------------------------------------------------------------
    def measure(self, genome) -> MeasuredTime:
        genome = tuple(int(b) for b in genome)
        low, res, slot = self._execute(genome)
        if low.failure is not None:
            return MeasuredTime.failed(low.failure)
        st = res.stats()
        st["slot"] = slot
        st["device"] = self.devices[slot]
        with self._count_lock:
            self.stats[genome] = st
            self.evaluations += 1
        if res.status == N.HP_OK:
            return MeasuredTime.ok(max(res.wall_s, 1e-9))
        if res.status == N.HP_TIMEOUT:
            return MeasuredTime.timeout()
        return MeasuredTime.failed(res.diag.decode(errors="replace") or f"status {res.status}")

    def run(self, genome, with_slot: bool = False, literal_gosa: bool = False):
        """Execute once and return the native result (raises on pattern failure);
        with_slot: (result, worker slot whose context holds the run's fields);
        literal_gosa: verification mode (HP_FLAG_LITERAL_GOSA, see run_for_output)."""
        genome = tuple(int(b) for b in genome)
        low, res, slot = self._execute(genome, N.FLAG_LITERAL_GOSA if literal_gosa else 0)
        if low.failure is not None:
            raise BaselineFailure(low.failure)
        if res.status != N.HP_OK:
            raise BaselineFailure(res.diag.decode(errors="replace"))
        with self._count_lock:
            self.stats[genome] = res.stats()
        return (res, slot) if with_slot else res

    def run_for_output(self, genome, literal_gosa: bool = True) -> str:
        """The program's stdout for this pattern (main's printf lines, evaluators.py:183-188).

        main prints its float gosa.  When the stencil's ss*ss terms are summed on the
        host that is the literal fp32 sequential sum.  When they are summed on the
        device, verification mode (``literal_gosa``, the default here: this is the
        verification path, not a fitness measurement) also writes the last
        iteration's terms out from the pattern's own device state and sums them in
        program order, so the printed value is comparable token for token with the
        original program's; with ``literal_gosa=False`` it is the fp32 rounding of
        the device's fp64 reduction (2.6 % off the sequential fp32 sum at M, which
        drifts: SURVEY.md §7.3)."""
        res = self.run(genome, literal_gosa=literal_gosa)
        lines = [f"{float(res.gosa_f32):.9e}"]
        lines += [f"{float(v):.9e}" for v in res.samples[:res.n_samples]]
        return "\n".join(lines) + "\n"

    def read_field(self, name: str, slot: Optional[int] = None, side: int = 0):
        """Host (side 0) or device (1) copy of a field after the last run in a worker slot
        (default: the slot of the most recent run -- pass the slot from
        ``run(..., with_slot=True)`` or ``stats[genome]["slot"]`` when measuring
        concurrently)."""
        if slot is None:
            with self._count_lock:
                slot = self._last_slot
        return self._context(slot).read_field(name, side)

    def close(self) -> None:
        with self._ctx_lock:
            for ctx in self._contexts.values():
                ctx.close()
            self._contexts.clear()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


def measure_baseline(evaluator, gene_len: int) -> float:
    """All-zero genome once, outside the GA (cli.py:200-208)."""
    m = evaluator.measure(tuple([0] * gene_len))
    if m.failure is not None:
        raise BaselineFailure(f"baseline run failed: {m.failure}")
    if m.timed_out:
        raise BaselineFailure("baseline run exceeded the timeout; "
                              "the unmodified program must complete")
    return m.seconds


def valid_genomes(loops, eligible_ids) -> list:
    """Genomes with no gene=1 loop nested inside another (272 of 8192 for Himeno)."""
    n = len(eligible_ids)
    out = []
    for value in range(1 << n):
        g = tuple((value >> (n - 1 - i)) & 1 for i in range(n))
        on = {lid for lid, b in zip(eligible_ids, g) if b}
        if not any(a in on for lid in on for a in loops.ancestors(lid)[1:]):
            out.append(g)
    return out
