"""Cost-model evaluator (reference-compatible) and its calibration from B200 measurements.

The reference ships a deterministic desk-scale evaluator that prices a genome as
overhead + per-loop CPU/GPU times + priced transfer events of its plan
(acctuner/evaluators.py:49-147; file format SPEC.md "CostModel file format").
This module keeps that API -- ``CostModel``, ``evaluate_costmodel``,
``CostModelEvaluator``, ``brute_force_optimum`` -- and adds ``calibrate``: a
least-squares fit of the model's per-loop times to measured B200 fitness runs
(SURVEY.md §8(f) rank 4), so the surrogate can pre-screen genomes and its
brute-force optimum can be compared with the measured one
(``scripts/calibrate_costmodel.py``).
"""

from __future__ import annotations

import json
from dataclasses import dataclass, field
from pathlib import Path
from typing import Optional

from .errors import EnumerationTooLarge, ModelIncomplete
from .evaluator import MeasuredTime
from .plan import Planner

BRUTE_FORCE_LIMIT = 20


@dataclass
class CostModel:
    overhead_s: float
    loop_cpu_s: dict
    loop_gpu_s: dict
    var_bytes: dict
    bandwidth_bytes_per_s: float
    latency_s: float
    note: str = ""

    def __post_init__(self):
        vals = [self.overhead_s, self.bandwidth_bytes_per_s, self.latency_s,
                *self.loop_cpu_s.values(), *self.loop_gpu_s.values(), *self.var_bytes.values()]
        if any(v < 0 for v in vals) or self.bandwidth_bytes_per_s == 0:
            raise ValueError("cost model components must be non-negative "
                             "with positive bandwidth")

    def transfer_event_s(self, var_name: str) -> float:
        if var_name not in self.var_bytes:
            raise ModelIncomplete(f"cost model has no bytes for variable {var_name!r}")
        return self.var_bytes[var_name] / self.bandwidth_bytes_per_s + self.latency_s

    @classmethod
    def from_json(cls, doc: dict) -> "CostModel":
        loops = doc.get("loops", {})
        return cls(overhead_s=float(doc.get("overhead_s", 0.0)),
                   loop_cpu_s={int(k): float(v["cpu_s"]) for k, v in loops.items()},
                   loop_gpu_s={int(k): float(v["gpu_s"]) for k, v in loops.items()},
                   var_bytes={k: float(v["bytes"]) for k, v in doc.get("vars", {}).items()},
                   bandwidth_bytes_per_s=float(doc["bandwidth_bytes_per_s"]),
                   latency_s=float(doc.get("latency_s", 0.0)), note=doc.get("note", ""))

    def to_json(self) -> dict:
        ids = sorted(set(self.loop_cpu_s) | set(self.loop_gpu_s))
        return {"overhead_s": self.overhead_s,
                "loops": {str(i): {"cpu_s": self.loop_cpu_s.get(i, 0.0),
                                   "gpu_s": self.loop_gpu_s.get(i, 0.0)} for i in ids},
                "vars": {k: {"bytes": v} for k, v in self.var_bytes.items()},
                "bandwidth_bytes_per_s": self.bandwidth_bytes_per_s,
                "latency_s": self.latency_s, "note": self.note}

    @classmethod
    def load(cls, path) -> "CostModel":
        return cls.from_json(json.loads(Path(path).read_text()))


def loop_modes(genome, loops, eligible_ids) -> dict:
    """Execution mode of every loop under a genome (nest-aware pricing).

    "gpu": outermost gene=1 loop of its chain (a device construct covering its subtree);
    "cpu": root of a subtree that runs entirely on the host; anything else ("covered",
    "driver": a host loop whose body launches device work, "inside": within a priced
    host subtree) costs nothing by itself.
    """
    gene = dict(zip(eligible_ids, genome))
    device = {l.loop_id for l in loops if gene.get(l.loop_id) == 1}
    modes = {}
    for l in loops:
        lid = l.loop_id
        chain = loops.ancestors(lid)
        if any(a in device for a in chain[1:]):
            modes[lid] = "covered"
        elif lid in device:
            modes[lid] = "gpu"
        else:
            sub_dev = any(lid in loops.ancestors(d)[1:] for d in device)
            parent = l.parent_loop
            if sub_dev:
                modes[lid] = "driver"
            elif parent is not None and modes.get(parent) == "driver":
                modes[lid] = "cpu"
            elif parent is None:
                modes[lid] = "cpu"
            else:
                modes[lid] = "inside"
    return modes


def evaluate_costmodel(genome, plan, model: CostModel, eligible_ids, refs,
                       loops=None) -> float:
    """overhead + CPU loops + GPU loops + priced static transfer events of the plan.

    Default: the reference's additive form (evaluators.py:94-105).  With ``loops`` the
    nest-aware form prices ``cpu_s`` for each host-only subtree root and ``gpu_s`` for
    each device anchor (see ``loop_modes``).
    """
    total = model.overhead_s
    if loops is None:
        for lid, bit in zip(eligible_ids, genome):
            table = model.loop_gpu_s if bit else model.loop_cpu_s
            if lid not in table:
                raise ModelIncomplete(f"cost model has no entry for loop {lid}")
            total += table[lid]
    else:
        for lid, mode in loop_modes(genome, loops, eligible_ids).items():
            if mode in ("cpu", "gpu"):
                table = model.loop_gpu_s if mode == "gpu" else model.loop_cpu_s
                if lid not in table:
                    raise ModelIncomplete(f"cost model has no entry for loop {lid}")
                total += table[lid]
    for entry in plan.entries:
        total += entry.events * model.transfer_event_s(refs.vars[entry.var].name)
    return total


class CostModelEvaluator:
    """Deterministic evaluator: plans transfers and prices the plan."""

    deterministic = True
    max_concurrency = 1

    def __init__(self, model: CostModel, loops, refs, eligible_ids, nest_aware: bool = False):
        self.model = model
        self.refs = refs
        self.loops = loops
        self.nest_aware = nest_aware
        self.eligible_ids = list(eligible_ids)
        self.planner = Planner(loops, refs, eligible_ids)

    def plan(self, genome):
        return self.planner.plan(genome)

    def measure(self, genome) -> MeasuredTime:
        plan = self.planner.plan(genome)
        return MeasuredTime.ok(evaluate_costmodel(
            genome, plan, self.model, self.eligible_ids, self.refs,
            self.loops if self.nest_aware else None))


def brute_force_optimum(model: CostModel, loops, refs, eligible_ids) -> tuple:
    """Exact minimiser over all 2^n genomes; ties go to the lowest binary value."""
    n = len(eligible_ids)
    if n > BRUTE_FORCE_LIMIT:
        raise EnumerationTooLarge(f"{n} genes exceed the 2^{BRUTE_FORCE_LIMIT} bound")
    planner = Planner(loops, refs, eligible_ids)
    best, best_t = None, float("inf")
    for value in range(1 << n):
        g = tuple((value >> (n - 1 - i)) & 1 for i in range(n))
        t = evaluate_costmodel(g, planner.plan(g), model, eligible_ids, refs)
        if t < best_t:
            best, best_t = g, t
    return best, best_t


# ---------------------------------------------------------------- calibration

def var_bytes_of(refs) -> dict:
    """Bytes moved by one transfer event of each plannable variable (fp32/int scalars)."""
    out = {}
    for v in refs.plannable():
        if v.extents:
            n = 1
            for e in v.extents:
                n *= int(e)
            out[v.name] = 4.0 * n
        else:
            out[v.name] = 8.0 if v.name == "gosa" else 4.0
    return out


@dataclass
class Calibration:
    model: CostModel
    residual_rms_s: float
    n_samples: int
    columns: list = field(default_factory=list)


def calibrate(samples, loops, refs, eligible_ids, bandwidth_bytes_per_s: float,
              latency_s: float, ridge: float = 1e-9, nest_aware: bool = False) -> Calibration:
    """Fit overhead and per-loop cpu_s / gpu_s to measured (genome, seconds) samples.

    The transfer term uses the plan's static events priced with the given bandwidth and
    latency (the reference model's form), and is subtracted before the non-negative
    least-squares fit of the loop terms (projected gradient on a ridge-regularised
    normal system; tiny and deterministic).
    """
    import numpy as np
    planner = Planner(loops, refs, eligible_ids)
    vb = var_bytes_of(refs)
    tmp = CostModel(0.0, {}, {}, vb, bandwidth_bytes_per_s, latency_s)
    n = len(eligible_ids)
    rows, ys = [], []
    for genome, seconds in samples:
        plan = planner.plan(genome)
        xfer = sum(e.events * tmp.transfer_event_s(refs.vars[e.var].name) for e in plan.entries)
        if nest_aware:
            modes = loop_modes(genome, loops, eligible_ids)
            x = [1.0] + [float(modes[l] == "cpu") for l in eligible_ids] \
                + [float(modes[l] == "gpu") for l in eligible_ids]
        else:
            x = [1.0] + [1.0 - b for b in genome] + [float(b) for b in genome]
        rows.append(x)
        ys.append(seconds - xfer)
    A = np.asarray(rows)
    y = np.asarray(ys)
    AtA = A.T @ A + ridge * np.eye(A.shape[1])
    Aty = A.T @ y
    theta = np.clip(np.linalg.lstsq(AtA, Aty, rcond=None)[0], 0.0, None)
    step = 1.0 / max(np.linalg.eigvalsh(AtA).max(), 1e-30)
    for _ in range(20000):                      # projected gradient: theta >= 0
        nxt = np.clip(theta - step * (AtA @ theta - Aty), 0.0, None)
        if np.max(np.abs(nxt - theta)) < 1e-15:
            theta = nxt
            break
        theta = nxt
    resid = A @ theta - y
    model = CostModel(overhead_s=float(theta[0]),
                      loop_cpu_s={lid: float(theta[1 + i]) for i, lid in enumerate(eligible_ids)},
                      loop_gpu_s={lid: float(theta[1 + n + i]) for i, lid in enumerate(eligible_ids)},
                      var_bytes=vb, bandwidth_bytes_per_s=bandwidth_bytes_per_s,
                      latency_s=latency_s,
                      note=f"calibrated on {len(samples)} B200 measurements (least squares"
                           f"{', nest-aware' if nest_aware else ''})")
    return Calibration(model, float(np.sqrt(np.mean(resid ** 2))), len(samples),
                       ["overhead"] + [f"cpu_{l}" for l in eligible_ids]
                       + [f"gpu_{l}" for l in eligible_ids])


def spearman(a, b) -> float:
    """Rank correlation (average ranks for ties)."""
    import numpy as np

    def ranks(x):
        x = np.asarray(x, dtype=float)
        order = np.argsort(x, kind="mergesort")
        r = np.empty(len(x))
        r[order] = np.arange(len(x), dtype=float)
        for v in np.unique(x):
            idx = np.where(x == v)[0]
            r[idx] = r[idx].mean()
        return r
    ra, rb = ranks(a), ranks(b)
    ra -= ra.mean()
    rb -= rb.mean()
    den = float(np.sqrt((ra ** 2).sum() * (rb ** 2).sum()))
    return float((ra * rb).sum() / den) if den else 0.0


def optimum_over(model: CostModel, loops, refs, eligible_ids, genomes,
                 nest_aware: bool = False) -> tuple:
    """Minimiser of the model over a given genome list (e.g. the runnable genomes)."""
    planner = Planner(loops, refs, eligible_ids)
    best, best_t = None, float("inf")
    for g in genomes:
        t = evaluate_costmodel(g, planner.plan(g), model, eligible_ids, refs,
                               loops if nest_aware else None)
        if t < best_t:
            best, best_t = g, t
    return best, best_t


def load_measurements(path) -> list:
    """(genome tuple, seconds) pairs from scripts/eval_all.py output."""
    out = []
    for line in Path(path).read_text().splitlines():
        d = json.loads(line)
        if d.get("summary") or not d.get("time_s"):
            continue
        out.append((tuple(int(c) for c in d["genome"]), float(d["time_s"])))
    return out
