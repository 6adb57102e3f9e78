"""Checkpoint / resume and per-evaluation records for a tuning run.

The reference keeps its ``EvalCache`` in memory only (``acctuner/ga.py:132-148``) and
writes its reports at the end (``cli.py:310-317``), so an interrupted search starts over.
``CheckpointedEvaluator`` wraps any evaluator plugin (the duck-typed ``measure`` /
``max_concurrency`` / ``deterministic`` interface, ``evaluators.py:124-128``) and appends
one JSON line per fresh measurement to a checkpoint file.  Restarted with the same file,
it answers the genomes already measured from the file instead of running them again.
Because ``run_ga`` is deterministic given the fitness values (``ga.py:183-265``: the
operators draw from the seeded RNG and the records are committed in genome order), a
resumed run replays the interrupted run's generations exactly and continues from where it
stopped -- the final records equal those of an uninterrupted run with the same
measurements.

Each line also carries the evaluation's metrics when the wrapped evaluator exposes them
(``B200Evaluator.stats``): device and worker slot, host / transfer / wall seconds,
H2D / D2H bytes and transfer counts, kernel launches, the achieved PCIe rate, and gosa.
"""

from __future__ import annotations

import json
import threading
from pathlib import Path

from .evaluator import MeasuredTime


def _key(genome) -> str:
    return "".join(str(int(b)) for b in genome)


class CheckpointedEvaluator:
    """Evaluator plugin that persists every fresh measurement and replays them."""

    def __init__(self, evaluator, path):
        self.inner = evaluator
        self.path = Path(path)
        self.max_concurrency = getattr(evaluator, "max_concurrency", 1) or 1
        self.deterministic = getattr(evaluator, "deterministic", False)
        self._lock = threading.Lock()
        self._known: dict = {}
        self.replayed = 0
        self.measured = 0
        if self.path.exists():
            for line in self.path.read_text().splitlines():
                if not line.strip():
                    continue
                rec = json.loads(line)
                self._known[rec["genome"]] = rec
        self.path.parent.mkdir(parents=True, exist_ok=True)

    def __getattr__(self, name):   # gene_length, plan, kinds, ... of the wrapped plugin
        return getattr(self.inner, name)

    @staticmethod
    def _to_measured(rec) -> MeasuredTime:
        if rec["outcome"] == "ok":
            return MeasuredTime.ok(rec["seconds"])
        if rec["outcome"] == "timeout":
            return MeasuredTime.timeout()
        return MeasuredTime.failed(rec.get("diagnostic") or "failed")

    def _record(self, genome, m: MeasuredTime) -> dict:
        rec = {"genome": _key(genome)}
        if m.timed_out:
            rec["outcome"] = "timeout"
        elif m.failure is not None:
            rec["outcome"] = "failed"
            rec["diagnostic"] = m.failure
        else:
            rec["outcome"] = "ok"
            rec["seconds"] = m.seconds
        st = getattr(self.inner, "stats", {}).get(tuple(int(b) for b in genome))
        if st and m.failure is None:
            xfer = st.get("xfer_s") or 0.0
            moved = (st.get("h2d_bytes") or 0) + (st.get("d2h_bytes") or 0)
            rec["metrics"] = {
                "device": st.get("device"), "slot": st.get("slot"),
                "wall_s": st.get("wall_s"), "host_s": st.get("host_s"), "xfer_s": xfer,
                "h2d_bytes": st.get("h2d_bytes"), "d2h_bytes": st.get("d2h_bytes"),
                "n_h2d": st.get("n_h2d"), "n_d2h": st.get("n_d2h"),
                "n_launch": st.get("n_launch"),
                "xfer_gbs": moved / xfer / 1e9 if xfer > 0 else None,
                "gosa": st.get("gosa")}
        return rec

    def measure(self, genome) -> MeasuredTime:
        key = _key(genome)
        with self._lock:
            rec = self._known.get(key)
            if rec is not None:
                self.replayed += 1
                return self._to_measured(rec)
        m = self.inner.measure(genome)
        rec = self._record(genome, m)
        with self._lock:
            if key not in self._known:
                self._known[key] = rec
                self.measured += 1
                with self.path.open("a") as fh:
                    fh.write(json.dumps(rec, sort_keys=True) + "\n")
                    fh.flush()
        return m

    def run_for_output(self, *a, **kw):
        return self.inner.run_for_output(*a, **kw)
