"""Checkpoint / resume of a tuning run (checkpoint.py): an interrupted GA resumed from its
checkpoint file ends with exactly the records of an uninterrupted run, re-measuring only
the genomes the interrupted run had not measured."""
import json
import random

import pytest

from paper_2002_12115_b200 import ga
from paper_2002_12115_b200.checkpoint import CheckpointedEvaluator
from paper_2002_12115_b200.evaluator import MeasuredTime


class TableEvaluator:
    """Deterministic fitness per genome; failures and timeouts for some; optionally dies
    after `die_after` measurements (the interruption)."""

    def __init__(self, gene_len, die_after=None, concurrency=1):
        self.gene_length = gene_len
        self.max_concurrency = concurrency
        self.calls = 0
        self.die_after = die_after
        self.stats = {}

    def measure(self, genome):
        self.calls += 1
        if self.die_after is not None and self.calls > self.die_after:
            raise KeyboardInterrupt("interrupted")
        key = "".join(map(str, genome))
        h = random.Random(key).random()
        if h < 0.1:
            return MeasuredTime.failed("nested compute construct")
        if h < 0.15:
            return MeasuredTime.timeout()
        return MeasuredTime.ok(0.001 + h)


def _records(res):
    return [r.to_json() for r in res.records], res.evaluations, res.best.genome


@pytest.mark.parametrize("concurrency", [1, 4])
def test_resume_reproduces_uninterrupted_run(tmp_path, concurrency):
    cfg = ga.GAConfig(population=10, generations=8, rng_seed=3)
    full = ga.run_ga(cfg, 13, TableEvaluator(13, concurrency=concurrency))
    ck = tmp_path / "evals.jsonl"
    first = TableEvaluator(13, die_after=25, concurrency=concurrency)
    with pytest.raises(KeyboardInterrupt):
        ga.run_ga(cfg, 13, CheckpointedEvaluator(first, ck))
    saved = [json.loads(l) for l in ck.read_text().splitlines()]
    assert 0 < len(saved) <= 25
    inner = TableEvaluator(13, concurrency=concurrency)
    wrapped = CheckpointedEvaluator(inner, ck)
    resumed = ga.run_ga(cfg, 13, wrapped)
    assert _records(resumed) == _records(full)
    assert wrapped.replayed == len(saved)
    assert inner.calls == full.evaluations - len(saved)
    # outcomes survive the round trip: failures and timeouts replay as such
    kinds = {r["outcome"] for r in (json.loads(l) for l in ck.read_text().splitlines())}
    assert "ok" in kinds
