"""Lower (genome, directive kinds, loop tree, TransferPlan) to a native hp_schedule.

This is the B200 replacement of the reference's emit step
(acctuner/emitter.py:132-228): instead of inserting pragma lines and
compiling, each plan entry becomes data-manager events attached to loop
statements, and each loop gets an execution kind.  The mapping follows the
emitted OpenACC's meaning:

=====================================  ===============================================
emitter output                         event(s)
=====================================  ===============================================
``declare create(x)`` (temp_region)    DECLARE(x) at program start      emitter.py:216-220
``update device(x)`` before open       UPDATE_DEVICE at (open loop, before)   221-224
``update self(x)`` after close         UPDATE_SELF at (close loop, after)     225-228
``data copyin/copyout/copy(x)`` { }    DATA_ENTER(copyin?) / DATA_EXIT(copyout?)  166-188
``data present(x)`` at a covered loop  PRESENT(x) at (site, before)           190-201
kind pragma on a gene=1 loop           loop_kind = directive kind             160-164
=====================================  ===============================================

Nested gene=1 loops: the reference emits a compute pragma on every gene=1
loop (emitter.py:160-164); nested compute constructs do not compile, so the
individual is penalised.  ``nested_policy="reject"`` (default) reproduces
that as ``MeasuredTime.failed`` before anything runs; ``"outermost"`` runs the
outermost anchor and treats inner genes as covered.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Optional

from . import native as N
from .errors import PlanInconsistent
from .kinds import DirectiveKind

NESTED_POLICIES = ("reject", "outermost")


@dataclass
class Lowered:
    """A schedule ready for hp_run, or the reason the pattern cannot run."""
    schedule: Optional[N.Schedule]
    failure: Optional[str] = None
    loop_kind: list = field(default_factory=list)
    events: list = field(default_factory=list)      # (loop, when, op, var, arg, entry)
    _keep: object = None                            # ctypes event array lifetime


def _nested_pairs(loops, gene: dict) -> list:
    out = []
    for l in loops:
        if gene.get(l.loop_id) != 1:
            continue
        for anc in loops.ancestors(l.loop_id)[1:]:
            if gene.get(anc) == 1:
                out.append((l.loop_id, anc))
                break
    return out


def loop_kinds(loops, gene: dict, kinds: dict, nested_policy: str = "reject",
               n_loops: int = N.NLOOPS):
    """Per-loop native kind, or (None, diagnostic) for a rejected pattern."""
    if nested_policy not in NESTED_POLICIES:
        raise ValueError(f"nested_policy must be one of {NESTED_POLICIES}")
    nested = _nested_pairs(loops, gene)
    if nested and nested_policy == "reject":
        inner, outer = nested[0]
        return None, (f"nested compute construct: loop {inner} ({kinds[inner].value}) "
                      f"inside gene=1 loop {outer} ({kinds[outer].value})")
    out = [N.K_HOST] * n_loops
    for l in loops:
        lid = l.loop_id
        anchor = None
        for a in reversed(loops.ancestors(lid)):
            if gene.get(a) == 1:
                anchor = a
                break
        if anchor is None:
            out[lid] = N.K_HOST
        elif anchor == lid:
            out[lid] = DirectiveKind(kinds[lid].value).native_code
        else:
            out[lid] = N.K_COVERED
    return out, None


def _loop_of_span(loops, file_id, span) -> int:
    for l in loops:
        if l.file_id == file_id and tuple(l.span) == tuple(span):
            return l.loop_id
    raise PlanInconsistent(f"plan span {span} in {file_id} is not a loop statement")


def plan_events(plan, loops, refs, gene: dict, var_id: dict = None) -> list:
    """TransferPlan entries -> ordered event tuples (loop, when, op, var, arg, entry).

    ``var_id`` maps plan variable keys to the executor's variable ids (default:
    the Himeno library's table)."""
    var_id = N.VAR_ID if var_id is None else var_id
    events = []
    declared = set()
    on = {lid for lid, bit in gene.items() if bit == 1}
    for idx, e in enumerate(plan.entries):
        for m in e.members:
            if m not in on:
                raise PlanInconsistent(f"plan covers loop {m} which is not gene=1")
        for site in e.present_sites:
            if site not in e.members:
                raise PlanInconsistent(f"present site {site} outside its region")
        key = e.var
        if key not in var_id:
            raise PlanInconsistent(f"variable {key!r} is not part of the program")
        var = var_id[key]
        open_loop = getattr(e, "open_loop", None)
        close_loop = getattr(e, "close_loop", None)
        if open_loop is None:
            open_loop = _loop_of_span(loops, e.open_file, e.open_span)
        if close_loop is None:
            close_loop = _loop_of_span(loops, e.close_file, e.close_span)
        into, out = e.direction.into_device, e.direction.out_of_device
        if e.temp_region:
            if var not in declared:
                declared.add(var)
                events.append((-1, N.BEFORE, N.EV_DECLARE, var, 0, idx))
            if into:
                events.append((open_loop, N.BEFORE, N.EV_UPDATE_DEVICE, var, 0, idx))
            if out:
                events.append((close_loop, N.AFTER, N.EV_UPDATE_SELF, var, 0, idx))
        else:
            events.append((open_loop, N.BEFORE, N.EV_DATA_ENTER, var, int(into), idx))
            events.append((close_loop, N.AFTER, N.EV_DATA_EXIT, var, int(out), idx))
        for site in e.present_sites:
            events.append((site, N.BEFORE, N.EV_PRESENT, var, 0, idx))
    return events


def lower(genome, eligible_ids, kinds: dict, loops, refs, plan, nn: int,
          flags: int, timeout_s: float = 180.0, nested_policy: str = "reject") -> Lowered:
    if len(genome) != len(eligible_ids):
        raise PlanInconsistent(f"genome length {len(genome)} != {len(eligible_ids)}")
    gene = {lid: int(b) for lid, b in zip(eligible_ids, genome)}
    lk, failure = loop_kinds(loops, gene, kinds, nested_policy)
    if failure is not None:
        return Lowered(None, failure)
    if nested_policy == "outermost":
        gene = {lid: int(lk[lid] not in (N.K_HOST, N.K_COVERED)) for lid in gene}
    events = plan_events(plan, loops, refs, gene) if plan is not None else []
    arr = (N.Event * max(1, len(events)))(*[N.Event(*ev) for ev in events])
    sched = N.Schedule()
    sched.n_loops = N.NLOOPS
    for lid in range(N.NLOOPS):
        sched.loop_kind[lid] = lk[lid]
    sched.n_events = len(events)
    sched.events = C.cast(arr, C.POINTER(N.Event))
    sched.nn = int(nn)
    sched.flags = int(flags)
    sched.timeout_s = float(timeout_s)
    return Lowered(sched, None, lk, events, arr)
