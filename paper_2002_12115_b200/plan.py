"""Per-genome CPU<->GPU transfer plan (the paper's batched/hoisted policy, §3.3).

Restates the reference planner (acctuner/transfer.py) over the duck-typed
model of ``model.py`` -- or a reference ``ProjectModel``: only ``loops``
(``get``/``ancestors``/iteration) and ``refs`` (``vars``/``order``/
``plannable``) are touched.  The plan is host-side metadata; it is computed
once per genome (and cached by the evaluator) and lowered to transfer events
that the native data manager executes (lower.py, csrc/executor.cpp).

Three stages, as in the reference (transfer.py:1-16, 413-418):

1. directions per (variable, gene=1 anchor)         ``plan_transfers``  (184-193)
2. batch consecutive anchors + hoist to the
   outermost legal loop, then demote partially
   overlapping structured regions                   ``hoist_and_batch`` (268-318),
                                                    ``_enforce_laminar`` (367-411)
3. globals -> device mirror (declare create/update) ``suppress_auto_transfers`` (322-329)

Output order and contents are identical to the reference for the same model
and genome; tests/test_plan_parity.py checks all 2^13 Himeno genomes.
"""

from __future__ import annotations

from dataclasses import dataclass, field, replace
from enum import Enum
from typing import Optional

from .errors import GenomeLengthMismatch


class Direction(Enum):
    COPYIN = "copyin"
    COPYOUT = "copyout"
    COPY = "copy"

    @property
    def into_device(self) -> bool:
        return self is not Direction.COPYOUT

    @property
    def out_of_device(self) -> bool:
        return self is not Direction.COPYIN

    @classmethod
    def of(cls, copyin: bool, copyout: bool) -> "Direction":
        if copyin and copyout:
            return cls.COPY
        return cls.COPYIN if copyin else cls.COPYOUT


@dataclass
class PlanEntry:
    """One data region for one variable (transfer.py:42-67)."""
    var: str
    direction: Direction
    members: list                  # gene=1 anchors covered, program order
    open_file: str
    open_span: tuple
    close_file: str
    close_span: tuple
    present_sites: list = field(default_factory=list)
    temp_region: bool = False
    open_loop: Optional[int] = None    # loop ids behind open/close spans (lowering aid)
    close_loop: Optional[int] = None

    @property
    def events(self) -> int:
        """Static transfer count of the entry (not the dynamic count)."""
        return int(self.direction.into_device) + int(self.direction.out_of_device)

    def to_json(self, refs) -> dict:
        return {"var": refs.vars[self.var].name, "direction": self.direction.value,
                "region_span": [self.open_span[0], self.close_span[1]],
                "present": list(self.present_sites), "temp_region": self.temp_region,
                "file": self.open_file}

    def signature(self) -> tuple:
        """Hashable identity used by parity tests."""
        return (self.var, self.direction.value, tuple(self.members), self.open_file,
                tuple(self.open_span), self.close_file, tuple(self.close_span),
                tuple(self.present_sites), self.temp_region)


@dataclass
class TransferPlan:
    entries: list = field(default_factory=list)

    def events_for(self, var: str) -> int:
        return sum(e.events for e in self.entries if e.var == var)

    def total_events(self) -> int:
        return sum(e.events for e in self.entries)

    def to_json(self, refs) -> list:
        return [e.to_json(refs) for e in self.entries]


@dataclass
class GpuRegionMap:
    """Gene=1 anchors grouped into runs not separated by a CPU write (transfer.py:84-96)."""
    runs: list
    gene: dict
    planner: "Planner"

    def run_of(self, loop_id: int) -> int:
        for idx, run in enumerate(self.runs):
            if loop_id in run:
                return idx
        raise KeyError(loop_id)


@dataclass
class _HostRef:
    order: int
    region: object
    read: bool
    written: bool
    defined: bool


@dataclass
class _DevUse:
    anchor: int
    order: int
    read: bool = False
    written: bool = False


class _Geometry:
    """Static facts of the loop tree, computed once per planner."""

    def __init__(self, loops, refs):
        self.loops = loops
        self.refs = refs
        ids = [l.loop_id for l in loops]
        self.chain = {i: list(loops.ancestors(i)) for i in ids}          # self -> outward
        self.outward_in = {i: list(reversed(c)) for i, c in self.chain.items()}
        self.parent = {l.loop_id: l.parent_loop for l in loops}
        self.file = {l.loop_id: l.file_id for l in loops}
        self.span = {l.loop_id: tuple(l.span) for l in loops}
        self.by_span = {(l.file_id, tuple(l.span)): l.loop_id for l in loops}
        self.pos = {i: refs.order(i) for i in ids}
        last = dict(self.pos)
        for i in ids:
            for a in self.chain[i]:
                if self.pos[i] > last[a]:
                    last[a] = self.pos[i]
        self.last = last                 # highest order inside each loop's subtree

    def anchor(self, region, gene) -> Optional[int]:
        """Outermost gene=1 loop whose subtree holds the region."""
        if not isinstance(region, int):
            return None
        for lid in self.outward_in[region]:
            if gene.get(lid) == 1:
                return lid
        return None

    def share_loop(self, region, anchor: int) -> bool:
        """Region and anchor sit under a common loop (a later iteration revisits both)."""
        if not isinstance(region, int):
            return False
        return not set(self.chain[region]).isdisjoint(self.chain[anchor])


class Planner:
    """Reusable planning context; ``plan(genome)`` is cheap per genome."""

    def __init__(self, loops, refs, eligible_ids):
        self.loops = loops
        self.refs = refs
        self.eligible_ids = list(eligible_ids)
        self._geo = _Geometry(loops, refs)
        self._vars = list(refs.plannable())

    # -- genome -----------------------------------------------------------------

    def gene_map(self, genome) -> dict:
        if len(genome) != len(self.eligible_ids):
            raise GenomeLengthMismatch(
                f"genome length {len(genome)} != eligible loops {len(self.eligible_ids)}")
        return {lid: int(bit) for lid, bit in zip(self.eligible_ids, genome)}

    # -- per-variable split into device uses and host references ---------------

    def _split(self, var, gene) -> tuple:
        geo = self._geo
        dev: dict = {}
        host = []
        for region, flags in var.refs.items():
            a = geo.anchor(region, gene)
            if a is None:
                host.append(_HostRef(self.refs.order(region), region,
                                     flags.read, flags.written, flags.defined))
                continue
            use = dev.get(a)
            if use is None:
                use = dev[a] = _DevUse(a, geo.pos[a])
            use.read |= flags.read
            use.written |= flags.written
        host.sort(key=lambda h: h.order)
        return sorted(dev.values(), key=lambda u: u.order), host

    def _before(self, h: _HostRef, use: _DevUse) -> bool:
        return h.order < use.order or self._geo.share_loop(h.region, use.anchor)

    def _after(self, h: _HostRef, use: _DevUse) -> bool:
        return h.order > use.order or self._geo.share_loop(h.region, use.anchor)

    # -- region representatives ---------------------------------------------------

    def _lift(self, group: list) -> list:
        """Member anchors lifted to their deepest common nesting level (transfer.py:197-216)."""
        paths = [self._geo.outward_in[u.anchor] for u in group]
        depth = 0
        while all(len(p) > depth for p in paths) and len({p[depth] for p in paths}) == 1:
            depth += 1
        if depth and any(len(p) == depth for p in paths):
            depth -= 1
        reps: list = []
        for p in paths:
            r = p[depth] if len(p) > depth else p[-1]
            if not reps or reps[-1] != r:
                reps.append(r)
        return reps

    def _make_entry(self, var, group: list, host: list, reps=None) -> Optional[PlanEntry]:
        first, last = group[0], group[-1]
        dev_reads = any(u.read for u in group)
        dev_writes = any(u.written for u in group)
        need_in = dev_reads and any((h.written or h.defined) and self._before(h, first)
                                    for h in host)
        need_out = dev_writes and any((h.read or h.written or h.defined) and self._after(h, last)
                                      for h in host)
        if not (need_in or need_out):
            return None
        if reps is None:
            reps = self._lift(group)
        geo = self._geo
        lo, hi = reps[0], reps[-1]
        anchors = [u.anchor for u in group]
        widened = len(group) > 1 or lo != group[0].anchor
        return PlanEntry(var.key, Direction.of(need_in, need_out), anchors,
                         geo.file[lo], geo.span[lo], geo.file[hi], geo.span[hi],
                         list(anchors) if widened else [], False, lo, hi)

    # -- stage 1 ------------------------------------------------------------------

    def plan_transfers(self, genome) -> TransferPlan:
        gene = self.gene_map(genome)
        out = []
        for var in self._vars:
            dev, host = self._split(var, gene)
            for use in dev:
                e = self._make_entry(var, [use], host)
                if e is not None:
                    out.append(e)
        return TransferPlan(out)

    # -- stage 2 ------------------------------------------------------------------

    def _blocks(self, h: _HostRef, dev_writes: bool) -> bool:
        return h.written or h.defined or (h.read and dev_writes)

    def _span_clear(self, start: int, end: int, host, dev_writes, foreign) -> bool:
        if any(start <= h.order <= end and self._blocks(h, dev_writes) for h in host):
            return False
        return not any(start <= u.order <= end for u in foreign)

    def _can_join(self, var, group: list, host: list, uses: list) -> bool:
        geo = self._geo
        reps = self._lift(group)
        start = min(geo.pos[r] for r in reps)
        end = max(geo.last[r] for r in reps)
        if geo.file[reps[0]] != geo.file[reps[-1]] and var.scope != "global":
            return False
        ids = {u.anchor for u in group}
        foreign = [u for u in uses if u.anchor not in ids]
        return self._span_clear(start, end, host, any(u.written for u in group), foreign)

    def _hoist(self, var, group: list, host: list, uses: list) -> list:
        """Move the region outward while the enclosing loop holds no other reference."""
        geo = self._geo
        reps = self._lift(group)
        ids = {u.anchor for u in group}
        foreign = [u for u in uses if u.anchor not in ids]
        dev_writes = any(u.written for u in group)
        while True:
            parents = {geo.parent[r] for r in reps}
            if len(parents) != 1:
                return reps
            parent = parents.pop()
            if parent is None:
                return reps
            if not self._span_clear(geo.pos[parent], geo.last[parent], host, dev_writes, foreign):
                return reps
            reps = [parent]

    def hoist_and_batch(self, plan: TransferPlan, regions: GpuRegionMap) -> TransferPlan:
        gene = regions.gene
        planned: dict = {}
        for e in plan.entries:
            planned.setdefault(e.var, set()).update(e.members)
        out = []
        for var in self._vars:
            if var.key not in planned:
                continue
            dev, host = self._split(var, gene)
            uses = [u for u in dev if u.anchor in planned[var.key]]
            groups: list = []
            for use in uses:
                if groups and self._can_join(var, groups[-1] + [use], host, uses):
                    groups[-1].append(use)
                else:
                    groups.append([use])
            for g in groups:
                e = self._make_entry(var, g, host, self._hoist(var, g, host, uses))
                if e is not None:
                    out.append(e)
        return TransferPlan(out)

    def _enforce_laminar(self, plan: TransferPlan, gene: dict) -> TransferPlan:
        """Structured (local) regions must nest; partial overlaps fall back to per-anchor."""
        def bounds(e):
            return e.open_span[0], e.close_span[1]

        def crosses(x, y) -> bool:
            if x.open_file != y.open_file:
                return False
            (s1, e1), (s2, e2) = bounds(x), bounds(y)
            if e1 <= s2 or e2 <= s1:
                return False
            return not (s1 <= s2 and e2 <= e1) and not (s2 <= s1 and e1 <= e2)

        local = [e for e in plan.entries if self.refs.vars[e.var].scope != "global"]
        kept: list = []
        dropped = set()
        for e in sorted(local, key=lambda e: bounds(e)[0] - bounds(e)[1]):
            if any(crosses(e, k) for k in kept):
                dropped.add(id(e))
            else:
                kept.append(e)
        if not dropped:
            return plan
        out = []
        for e in plan.entries:
            if id(e) not in dropped:
                out.append(e)
                continue
            var = self.refs.vars[e.var]
            dev, host = self._split(var, gene)
            for use in dev:
                if use.anchor in e.members:
                    single = self._make_entry(var, [use], host)
                    if single is not None:
                        out.append(single)
        return TransferPlan(out)

    # -- stage 3 ------------------------------------------------------------------

    def suppress_auto_transfers(self, plan: TransferPlan) -> TransferPlan:
        return TransferPlan([
            replace(e, temp_region=self.refs.vars[e.var].scope == "global",
                    members=list(e.members), present_sites=list(e.present_sites))
            for e in plan.entries])

    # -- chain --------------------------------------------------------------------

    def compute_gpu_regions(self, genome, plan: TransferPlan) -> GpuRegionMap:
        """Anchors in program order, split where a host write to a planned var intervenes."""
        gene = self.gene_map(genome)
        geo = self._geo
        anchors = sorted({a for l in self.loops
                          if (a := geo.anchor(l.loop_id, gene)) is not None},
                         key=lambda a: geo.pos[a])
        host_writes = []
        for key in {e.var for e in plan.entries}:
            for region, flags in self.refs.vars[key].refs.items():
                if geo.anchor(region, gene) is None and (flags.written or flags.defined):
                    host_writes.append(self.refs.order(region))
        runs: list = []
        for a in anchors:
            if runs and not any(geo.pos[runs[-1][-1]] < w < geo.pos[a] for w in host_writes):
                runs[-1].append(a)
            else:
                runs.append([a])
        anchor_set = set(anchors)
        for l in self.loops:
            lid = l.loop_id
            if gene.get(lid) == 1 and lid not in anchor_set:
                a = geo.anchor(lid, gene)
                for run in runs:
                    if a in run:
                        run.append(lid)
                        break
        return GpuRegionMap(runs, gene, self)

    def plan(self, genome) -> TransferPlan:
        raw = self.plan_transfers(genome)
        regions = self.compute_gpu_regions(genome, raw)
        batched = self._enforce_laminar(self.hoist_and_batch(raw, regions), regions.gene)
        return self.suppress_auto_transfers(batched)


# -- module-level surface (transfer.py:425-454) ---------------------------------------

def plan_transfers(genome, loops, refs, eligible_ids) -> TransferPlan:
    return Planner(loops, refs, eligible_ids).plan_transfers(genome)


def compute_gpu_regions(genome, loops, refs, eligible_ids, plan) -> GpuRegionMap:
    return Planner(loops, refs, eligible_ids).compute_gpu_regions(genome, plan)


def hoist_and_batch(plan: TransferPlan, regions: GpuRegionMap) -> TransferPlan:
    return regions.planner.hoist_and_batch(plan, regions)


def suppress_auto_transfers(plan: TransferPlan, refs, planner=None) -> TransferPlan:
    return TransferPlan([
        replace(e, temp_region=refs.vars[e.var].scope == "global",
                members=list(e.members), present_sites=list(e.present_sites))
        for e in plan.entries])


def plan_for_genome(genome, loops, refs, eligible_ids) -> TransferPlan:
    return Planner(loops, refs, eligible_ids).plan(genome)
