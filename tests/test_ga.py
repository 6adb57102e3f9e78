"""GA parity with the reference (bit-exact streams) and SPEC.md known answers."""
import hashlib
import json
import random

import pytest

from conftest import GOLDEN
from paper_2002_12115_b200 import ga
from paper_2002_12115_b200.errors import FitnessDomainError, LengthMismatch, ZeroGeneLength
from paper_2002_12115_b200.evaluator import MeasuredTime


def replay_time(genome):
    # identical to oracle/pin_reference.py::replay_time
    h = int(hashlib.sha256("".join(map(str, genome)).encode()).hexdigest()[:12], 16)
    if h % 17 == 0:
        return MeasuredTime.failed("replay: compile failed")
    if h % 23 == 0:
        return MeasuredTime.timeout()
    return MeasuredTime.ok(0.05 + (h % 100000) / 1000.0)


class Replay:
    deterministic = True

    def __init__(self, width=1):
        self.max_concurrency = width
        self.calls = []

    def measure(self, genome):
        self.calls.append(genome)
        return replay_time(genome)


@pytest.mark.parametrize("width", [1, 8])
def test_streams_bit_exact_with_reference(width):
    streams = json.loads((GOLDEN / "ga_streams.json").read_text())
    assert len(streams) == 12
    for s in streams:
        res = ga.run_ga(ga.GAConfig(**s["config"]), s["gene_len"], Replay(width))
        assert res.evaluations == s["evaluations"]
        assert res.best.to_json() == s["best"]
        assert [r.to_json() for r in res.records] == s["records"]


def test_first_genome_seed0():
    # random.Random(0) -> first genome 1101111110010
    pop = ga.init_population(13, 10, random.Random(0))
    assert ga.genome_str(pop[0]) == "1101111110010"
    assert len(pop) == 10 and all(len(g) == 13 for g in pop)


def test_fitness_law():
    assert ga.fitness(1.0) == 1.0
    # SPEC.md:328 prints 0.178744...; 31.3**-0.5 = 0.1787425 (the SPEC rounds loosely)
    assert abs(ga.fitness(31.3) - 0.178744) < 2e-6
    assert abs(ga.fitness(1000) - 0.0316228) < 1e-7
    for t in (0.001, 1, 31.3, 1000):
        assert abs(ga.fitness(t) - t ** -0.5) < 1e-12
    with pytest.raises(FitnessDomainError):
        ga.fitness(0)


def test_roulette_probabilities():
    inds = [ga.Individual((0,), 1.0, 0.3, "fresh"), ga.Individual((1,), 1.0, 0.1, "fresh")]
    rng = random.Random(7)
    hits = sum(ga.roulette_pick(inds, rng).genome == (0,) for _ in range(20000))
    assert abs(hits / 20000 - 0.75) < 0.02


def test_crossover_and_mutation_kats():
    class Fixed:
        def random(self):
            return 0.0

        def randint(self, a, b):
            return 2
    assert ga.crossover((1, 1, 1, 1), (0, 0, 0, 0), 0.9, Fixed()) == ((1, 1, 0, 0), (0, 0, 1, 1))
    assert ga.crossover((1, 0, 1), (0, 1, 1), 0.0, random.Random(1)) == ((1, 0, 1), (0, 1, 1))
    with pytest.raises(LengthMismatch):
        ga.crossover((1,), (0, 0), 0.5, random.Random(1))
    g = (1, 0, 1, 1, 0)
    assert ga.mutate(g, 0.0, random.Random(3)) == g
    assert ga.mutate(g, 1.0, random.Random(3)) == tuple(1 - b for b in g)
    rng = random.Random(11)
    flips = sum(sum(ga.mutate((0,) * 100, 0.05, rng)) for _ in range(1000))
    assert 0.045 <= flips / 1e5 <= 0.055


def test_cache_and_penalties():
    ev = Replay()
    cache = ga.EvalCache()
    a = ga.evaluate_with_cache((1, 0, 1), ev, cache, 1000.0)
    b = ga.evaluate_with_cache((1, 0, 1), ev, cache, 1000.0)
    assert len(ev.calls) == 1 and b.eval_source == "cache" and a.time_s == b.time_s

    class Bad:
        def measure(self, g):
            return MeasuredTime.failed("boom") if g[0] else MeasuredTime.timeout()
    c = ga.evaluate_with_cache((1,), Bad(), ga.EvalCache(), 1000.0)
    assert c.time_s == 1000.0 and c.eval_source == "penalty"
    d = ga.evaluate_with_cache((0,), Bad(), ga.EvalCache(), 1000.0)
    assert d.time_s == 1000.0 and d.timed_out and d.eval_source == "fresh"
    assert d.fitness == ga.fitness(1000.0)


def test_elitism_monotone_and_population_constant():
    for seed in range(20):
        res = ga.run_ga(ga.GAConfig(population=9, generations=8, rng_seed=seed), 13, Replay())
        best = [r.best_time_s for r in res.records]
        assert all(b2 <= b1 for b1, b2 in zip(best, best[1:]))
        assert all(len(r.individuals) == 9 for r in res.records)


def test_zero_gene_length():
    with pytest.raises(ZeroGeneLength):
        ga.init_population(0, 4, random.Random(0))


def test_config_validation():
    with pytest.raises(ValueError):
        ga.GAConfig(population=0)
    with pytest.raises(ValueError):
        ga.GAConfig(elitism_count=10, population=10)
    cfg = ga.GAConfig.from_json({"population": 20, "generations": 3, "unknown": 1})
    assert cfg.population == 20 and cfg.generations == 3
