"""Generated B200 executors (codegen.py) behind the reference's evaluator plugin API.

``GenEvaluator(app)`` is the drop-in for ``ExternalEvaluator`` (acctuner/
evaluators.py:168-222) on any application with a generated executor
(``APPS``: NAS FT classes S / W, and Himeno XS as a cross-check of the
hand-written library): ``measure(genome) -> MeasuredTime``, ``max_concurrency``
(worker slots = devices x workers_per_device, one context each),
``deterministic = False`` and ``run_for_output`` for ``verify_results``
(cli.py:155-186).  Per genome: ``Planner.plan`` (plan.py, the reference's
planner) -> ``lower`` (lower.py, the same event semantics as the Himeno
library) -> ``hpg_run`` of ``libapp_<app>.so`` (include/app_b200.h).
"""

from __future__ import annotations

import ctypes as C
import queue
import threading
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass
from pathlib import Path
from typing import Optional

from . import native as N
from .errors import (BaselineFailure, ConfigError, DeviceError, EvaluatorUnavailable,
                     NativeUnavailable)
from .evaluator import MeasuredTime, TRANSFER_MODES
from .lower import NESTED_POLICIES, loop_kinds, plan_events
from .plan import Planner

LIB_DIR = Path(__file__).resolve().parent / "_native"


@dataclass(frozen=True)
class AppSpec:
    name: str
    text: object          # () -> program text
    program: object       # () -> object with .model / .eligible / .kinds
    verify: object = None  # stdout -> bool (application's own correctness check)


def _ft_spec(cls):
    from .apps import ft
    return AppSpec(f"ft_{cls.lower()}", lambda: ft.source_text(cls), lambda: ft.program(cls),
                   lambda out: ft.checksum_error(out, cls) <= 1e-9)


def _himeno_spec():
    from .apps import himeno
    return AppSpec("himeno_xs", lambda: himeno.source_text(himeno.size("XS"), 3),
                   himeno.program)


def app_specs() -> dict:
    return {s.name: s for s in (_ft_spec("S"), _ft_spec("W"), _ft_spec("A"), _himeno_spec())}


APPS = ("ft_s", "ft_w", "ft_a", "himeno_xs")


class Event(C.Structure):
    _fields_ = [("loop_id", C.c_int32), ("when", C.c_int32), ("op", C.c_int32),
                ("var", C.c_int32), ("arg", C.c_int32), ("entry", C.c_int32)]


class Schedule(C.Structure):
    _fields_ = [("n_loops", C.c_int32), ("loop_kind", C.POINTER(C.c_int32)),
                ("n_events", C.c_int32), ("events", C.POINTER(Event)),
                ("flags", C.c_int32), ("timeout_s", C.c_double)]


class Result(C.Structure):
    _fields_ = [("wall_s", C.c_double), ("xfer_s", C.c_double),
                ("h2d_bytes", C.c_uint64), ("d2h_bytes", C.c_uint64),
                ("n_h2d", C.c_uint64), ("n_d2h", C.c_uint64),
                ("n_skipped_stale", C.c_uint64), ("n_implicit", C.c_uint64),
                ("n_launch", C.c_uint64), ("n_guard_init", C.c_uint64),
                ("status", C.c_int32), ("diag", C.c_char * 256)]

    def stats(self) -> dict:
        return {"wall_s": self.wall_s, "xfer_s": self.xfer_s, "h2d_bytes": self.h2d_bytes,
                "d2h_bytes": self.d2h_bytes, "n_h2d": self.n_h2d, "n_d2h": self.n_d2h,
                "n_skipped_stale": self.n_skipped_stale, "n_implicit": self.n_implicit,
                "n_launch": self.n_launch, "n_guard_init": self.n_guard_init,
                "status": self.status,
                "diag": self.diag.decode(errors="replace")}


FLAG_GUARD, FLAG_FRESH = 1, 2

SIGNATURES = {
    "hpg_create": (C.c_int, [C.c_int, C.POINTER(C.c_void_p)]),
    "hpg_destroy": (None, [C.c_void_p]),
    "hpg_run": (C.c_int, [C.c_void_p, C.POINTER(Schedule), C.POINTER(Result)]),
    "hpg_output": (C.c_size_t, [C.c_void_p, C.c_char_p, C.c_size_t]),
    "hpg_n_loops": (C.c_int, []),
    "hpg_n_vars": (C.c_int, []),
    "hpg_var_name": (C.c_char_p, [C.c_int]),
    "hpg_loop_kind": (C.c_int, [C.c_int]),
    "hpg_loop_note": (C.c_char_p, [C.c_int]),
    "hpg_last_error": (C.c_char_p, []),
}

_LIBS: dict = {}
_LIB_LOCK = threading.Lock()


def lib_path(app: str) -> Path:
    return LIB_DIR / f"libapp_{app}.so"


class AppLib:
    """One generated executor library: loop / variable tables and the C ABI."""

    def __init__(self, app: str):
        path = lib_path(app)
        if not path.exists():
            raise NativeUnavailable(f"{path.name} is not built (python -m "
                                    f"paper_2002_12115_b200.build): no CPU fallback exists")
        self.app = app
        self.lib = C.CDLL(str(path))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(self.lib, name)
            fn.restype, fn.argtypes = res, args
        self.n_loops = self.lib.hpg_n_loops()
        self.var_names = [self.lib.hpg_var_name(v).decode() for v in range(self.lib.hpg_n_vars())]
        self.var_id = {n: v for v, n in enumerate(self.var_names)}
        self.loop_notes = [self.lib.hpg_loop_note(l).decode() for l in range(self.n_loops)]

    def last_error(self) -> str:
        e = self.lib.hpg_last_error()
        return e.decode(errors="replace") if e else ""


def load(app: str) -> AppLib:
    with _LIB_LOCK:
        if app not in _LIBS:
            _LIBS[app] = AppLib(app)
        return _LIBS[app]


class GenContext:
    """One executor context (device < 0: host only)."""

    def __init__(self, app: AppLib, device: int):
        self.app = app
        self.ptr = C.c_void_p()
        rc = app.lib.hpg_create(int(device), C.byref(self.ptr))
        if rc != 0:
            raise DeviceError(f"hpg_create({device}) for {app.app}: {app.last_error()} "
                                f"(rc={rc})")

    def run(self, sched: Schedule) -> Result:
        res = Result()
        rc = self.app.lib.hpg_run(self.ptr, C.byref(sched), C.byref(res))
        if rc < 0:
            raise EvaluatorUnavailable(f"hpg_run: {self.app.last_error()} (rc={rc})")
        return res

    def output(self) -> str:
        n = self.app.lib.hpg_output(self.ptr, None, 0)
        buf = C.create_string_buffer(n + 1)
        self.app.lib.hpg_output(self.ptr, buf, n + 1)
        return buf.value.decode()

    def close(self):
        if self.ptr:
            self.app.lib.hpg_destroy(self.ptr)
            self.ptr = C.c_void_p()


@dataclass
class GenLowered:
    schedule: Optional[Schedule]
    failure: Optional[str] = None
    loop_kind: list = None
    events: list = None
    _keep: tuple = ()


def lower(genome, eligible_ids, kinds: dict, loops, plan, app: AppLib, flags: int,
          timeout_s: float = 180.0, nested_policy: str = "reject") -> GenLowered:
    if len(genome) != len(eligible_ids):
        raise ConfigError(f"genome length {len(genome)} != {len(eligible_ids)}")
    gene = {lid: int(b) for lid, b in zip(eligible_ids, genome)}
    lk, failure = loop_kinds(loops, gene, kinds, nested_policy, app.n_loops)
    if failure is not None:
        return GenLowered(None, failure)
    if nested_policy == "outermost":
        gene = {lid: int(lk[lid] not in (N.K_HOST, N.K_COVERED)) for lid in gene}
    events = plan_events(plan, loops, None, gene, app.var_id) if plan is not None else []
    ev = (Event * max(1, len(events)))(*[Event(*e) for e in events])
    kinds_arr = (C.c_int32 * app.n_loops)(*lk)
    sched = Schedule(app.n_loops, C.cast(kinds_arr, C.POINTER(C.c_int32)), len(events),
                     C.cast(ev, C.POINTER(Event)), int(flags), float(timeout_s))
    return GenLowered(sched, None, lk, events, (ev, kinds_arr))


class GenEvaluator:
    """Fitness of gene patterns of a generated application on B200s (plugin API)."""

    deterministic = False

    def __init__(self, app: str = "ft_s", devices=None, *, transfer_mode: str = "batched",
                 nested_policy: str = "reject", coherence_guard: bool = True,
                 fresh_process: bool = True, timeout_s: float = 180.0,
                 workers_per_device: int = 1, verify_each: bool = False, genes=None):
        specs = app_specs()
        if app not in specs:
            raise ConfigError(f"no generated executor for {app!r} (one of {sorted(specs)})")
        if transfer_mode not in TRANSFER_MODES:
            raise ConfigError(f"transfer_mode must be one of {TRANSFER_MODES}")
        if nested_policy not in NESTED_POLICIES:
            raise ConfigError(f"nested_policy must be one of {NESTED_POLICIES}")
        self.spec = specs[app]
        prog = self.spec.program()
        self.loops, self.refs = prog.model.loops, prog.model.refs
        self.eligible_ids = list(prog.eligible)
        self.classified_ids = list(prog.eligible)
        self.kinds = dict(prog.kinds)
        self.lib = load(app)
        if self.lib.n_loops != len(self.loops):
            raise NativeUnavailable(f"{app}: library has {self.lib.n_loops} loops, "
                                    f"model {len(self.loops)} (rebuild)")
        self.transfer_mode = transfer_mode
        self.nested_policy = nested_policy
        self.timeout_s = float(timeout_s)
        self.flags = (FLAG_GUARD if coherence_guard else 0) | (FLAG_FRESH if fresh_process else 0)
        devices = [0] if devices is None else list(devices)
        self.devices = devices * max(1, int(workers_per_device))
        if not self.devices:
            raise EvaluatorUnavailable("no devices to evaluate on")
        self.max_concurrency = len(self.devices)
        self._contexts: dict = {}
        self._ctx_lock = threading.Lock()
        self._free: "queue.Queue[int]" = queue.Queue()
        for slot in range(len(self.devices)):
            self._free.put(slot)
        self._lowered: dict = {}
        self._low_lock = threading.Lock()
        self.stats: dict = {}
        self.outputs: dict = {}
        self.evaluations = 0
        # verify_each: every run's stdout is checked against the all-CPU program's with
        # the reference's verify_results rule (cli.py:155-186); a pattern whose device
        # execution changes the result (a false accept of the static probe, e.g. a
        # parallel loop over a scalar-carried chain) is returned as failed, so the GA
        # searches correct patterns only.  Off by default: the reference verifies only
        # the final best pattern.
        self.verify_each = bool(verify_each)
        self._baseline_out: Optional[str] = None
        self.planner = Planner(self.loops, self.refs, self.eligible_ids)
        self.probe_log: dict = {}
        self.probe_times: dict = {}     # loop id (or "cpu") -> best single-gene wall seconds
        genes_arg = genes
        if genes in ("verified", "screened"):
            genes = self.verified_loops()
            if genes_arg == "screened":
                # the paper's narrowing of the search space: keep the loops whose device
                # version alone does not slow the program down (within 5 %)
                cpu = self.probe_times.get("cpu")
                genes = [l for l in genes if self.probe_times[l] <= 1.05 * cpu]
        if genes is not None:
            # restrict the genome to a subset of the classified loops (gene order kept)
            keep = set(int(g) for g in genes)
            unknown = keep - set(self.classified_ids)
            if unknown:
                raise ConfigError(f"loops {sorted(unknown)} are not eligible")
            self.eligible_ids = [l for l in self.classified_ids if l in keep]
            self.planner = Planner(self.loops, self.refs, self.eligible_ids)
            with self._low_lock:
                self._lowered.clear()

    @property
    def gene_length(self) -> int:
        return len(self.eligible_ids)

    def plan(self, genome):
        genome = tuple(int(b) for b in genome)
        if self.transfer_mode == "batched":
            return self.planner.plan(genome)
        return self.planner.plan_transfers(genome)

    def lowered(self, genome) -> GenLowered:
        genome = tuple(int(b) for b in genome)
        with self._low_lock:
            low = self._lowered.get(genome)
        if low is None:
            self.planner.gene_map(genome)
            low = lower(genome, self.eligible_ids, self.kinds, self.loops, self.plan(genome),
                        self.lib, self.flags, self.timeout_s, self.nested_policy)
            with self._low_lock:
                self._lowered[genome] = low
        return low

    def _context(self, slot: int) -> GenContext:
        with self._ctx_lock:
            ctx = self._contexts.get(slot)
            if ctx is None:
                ctx = GenContext(self.lib, self.devices[slot])
                self._contexts[slot] = ctx
            return ctx

    def prepare(self) -> None:
        missing = [s for s in range(len(self.devices)) if s not in self._contexts]
        if missing:
            with ThreadPoolExecutor(max_workers=len(missing)) as pool:
                list(pool.map(self._context, missing))

    def _execute(self, genome):
        low = self.lowered(genome)
        if low.failure is not None:
            return low, None, None
        slot = self._free.get()
        try:
            ctx = self._context(slot)
            res = ctx.run(low.schedule)
            out = ctx.output()
        finally:
            self._free.put(slot)
        return low, res, out

    def measure(self, genome) -> MeasuredTime:
        genome = tuple(int(b) for b in genome)
        low, res, out = self._execute(genome)
        if low.failure is not None:
            return MeasuredTime.failed(low.failure)
        self.stats[genome] = res.stats()
        self.outputs[genome] = out
        self.evaluations += 1
        if res.status == N.HP_OK:
            if self.verify_each and any(genome):
                from .tune import verify_results
                rep = verify_results(self.baseline_output(), out)
                if not rep.passed:
                    return MeasuredTime.failed("result differs from the all-CPU program: "
                                               + "; ".join(rep.detail[:2]))
            return MeasuredTime.ok(max(res.wall_s, 1e-9))
        if res.status == N.HP_TIMEOUT:
            return MeasuredTime.timeout()
        return MeasuredTime.failed(res.diag.decode(errors="replace") or f"status {res.status}")

    def verified_loops(self, trials: int = 2) -> list:
        """Eligibility probe of the generated executor (the B200 analogue of the
        reference's compile probe, classify.py:234-274), for every classified loop:

        * static: a ``parallel loop`` / ``parallel loop vector`` with a loop-carried
          scalar, or any loop whose iterations write the same array elements (an
          output dependence, ``codegen.shared_writes``), is rejected -- the static
          probe (classify.py:200-231) only looks at subscripts that use the index;
        * execution: the loop alone on the GPU under its kind, ``trials`` runs, each
          stdout checked against the all-CPU program's with verify_results.

        ``probe_log`` keeps the reason per loop."""
        from . import codegen
        from .tune import verify_results
        prog = codegen.CProgram(self.spec.text())
        base = self.baseline_output()
        zero = tuple(0 for _ in self.classified_ids)
        zlow = lower(zero, list(self.classified_ids), self.kinds, self.loops,
                     Planner(self.loops, self.refs, list(self.classified_ids)).plan(zero), self.lib,
                     self.flags, self.timeout_s, self.nested_policy)
        ctimes = []
        for _ in range(max(1, trials)):
            slot = self._free.get()
            try:
                ctimes.append(self._context(slot).run(zlow.schedule).wall_s)
            finally:
                self._free.put(slot)
        self.probe_times["cpu"] = min(ctimes)
        ok = []
        full = list(self.classified_ids)
        full_planner = Planner(self.loops, self.refs, full)
        for lid in full:
            loop = self.loops.get(lid)
            kind = self.kinds[lid].value
            kp = codegen.plan_kernel(prog, loop, kind, self.loops)
            if kp is not None and kp.carried and kind != "kernels":
                self.probe_log[lid] = ("loop-carried scalar " + ", ".join(d.name for d in kp.carried)
                                       + f" under {kind}")
                continue
            shared = codegen.shared_writes(prog, loop)
            if shared:
                self.probe_log[lid] = "iterations write the same elements of " + ", ".join(shared)
                continue
            g = tuple(int(l == lid) for l in full)
            low = lower(g, full, self.kinds, self.loops, full_planner.plan(g), self.lib,
                        self.flags, self.timeout_s, self.nested_policy)
            verdict = None
            best = float("inf")
            for _ in range(max(1, trials)):
                slot = self._free.get()
                try:
                    ctx = self._context(slot)
                    res = ctx.run(low.schedule)
                    out = ctx.output()
                finally:
                    self._free.put(slot)
                if res.status != N.HP_OK:
                    verdict = f"run failed: {res.diag.decode(errors='replace')}"
                    break
                rep = verify_results(base, out)
                if not rep.passed:
                    verdict = "result differs: " + "; ".join(rep.detail[:1])
                    break
                best = min(best, res.wall_s)
            if verdict is None:
                ok.append(lid)
                self.probe_times[lid] = best
                verdict = f"verified ({self.lib.loop_notes[lid]}, {res.wall_s * 1e3:.1f} ms)"
            self.probe_log[lid] = verdict
        return ok

    def baseline_output(self) -> str:
        """stdout of the all-CPU pattern (computed once)."""
        if self._baseline_out is None:
            self._baseline_out = self.run_for_output((0,) * self.gene_length)
        return self._baseline_out

    def run_for_output(self, genome) -> str:
        genome = tuple(int(b) for b in genome)
        low, res, out = self._execute(genome)
        if low.failure is not None:
            raise BaselineFailure(low.failure)
        if res.status != N.HP_OK:
            raise BaselineFailure(res.diag.decode(errors="replace"))
        return out

    def close(self) -> None:
        with self._ctx_lock:
            for ctx in self._contexts.values():
                ctx.close()
            self._contexts.clear()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()
