"""Genetic search over offload genomes (paper §3.2/§5.1.2), driving the evaluator.

The GA is host logic around the hot path: every fresh genome becomes one
``evaluator.measure`` call (one application run on a B200).  Operators are
*bit-exact* with the reference (acctuner/ga.py): one ``random.Random(seed)``
is consumed in the reference call order:

* init (ga.py:95-101): ``randint(0, 1)`` per bit, genome by genome;
* per next generation (ga.py:248-265): elites (no RNG) then per pair
  ``random()`` x2 (roulette, ga.py:104-112), ``random()`` (+ ``randint(1, n-1)``
  when crossing, ga.py:115-124), ``random()`` per bit x2 (mutation,
  ga.py:127-129); an odd last slot is roulette + mutation.

Fresh genomes of one generation are measured concurrently up to
``evaluator.max_concurrency`` (one per B200 for ``B200Evaluator``) and
committed in genome order, so the records do not depend on completion order
(ga.py:214-245).
"""

from __future__ import annotations

import bisect
import random
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass
from typing import Callable, Optional

from .errors import FitnessDomainError, LengthMismatch, ZeroGeneLength

Genome = tuple


def fitness(time_s: float) -> float:
    """time^(-1/2) (paper §5.1.2); undefined for non-positive times."""
    if time_s <= 0:
        raise FitnessDomainError(f"fitness undefined for time {time_s!r}")
    return time_s ** -0.5


@dataclass
class GAConfig:
    population: int = 10
    generations: int = 10
    crossover_rate: float = 0.9
    mutation_rate: float = 0.05
    timeout_s: float = 180.0
    penalty_time_s: float = 1000.0
    rng_seed: int = 0
    elitism_count: int = 1

    def __post_init__(self):
        if self.population < 1 or self.generations < 1:
            raise ValueError("population and generations must be positive")
        for name in ("crossover_rate", "mutation_rate"):
            if not 0.0 <= getattr(self, name) <= 1.0:
                raise ValueError(f"{name} outside [0, 1]")
        if not 0 <= self.elitism_count < self.population:
            raise ValueError("elitism_count must be in [0, population)")

    @classmethod
    def from_json(cls, doc: dict) -> "GAConfig":
        known = cls.__dataclass_fields__  # type: ignore[attr-defined]
        return cls(**{k: v for k, v in doc.items() if k in known})


@dataclass(frozen=True)
class Individual:
    genome: Genome
    time_s: float            # effective: penalty already applied
    fitness: float
    eval_source: str         # "fresh" | "cache" | "penalty"
    timed_out: bool = False
    diagnostic: str = ""

    def to_json(self) -> dict:
        return {"genome": genome_str(self.genome), "time_s": self.time_s,
                "fitness": self.fitness, "eval_source": self.eval_source,
                "timed_out": self.timed_out}


@dataclass
class GenerationRecord:
    generation: int
    individuals: list
    best_genome: Genome       # best so far over the run
    best_time_s: float

    def to_json(self) -> dict:
        return {"generation": self.generation,
                "individuals": [i.to_json() for i in self.individuals],
                "best_genome": genome_str(self.best_genome),
                "best_time_s": self.best_time_s}


def genome_str(genome: Genome) -> str:
    return "".join(map(str, genome))


def genome_from_str(text: str) -> Genome:
    return tuple(int(ch) for ch in text)


def init_population(gene_len: int, m: int, rng: random.Random) -> list:
    if gene_len < 1:
        raise ZeroGeneLength("no eligible loops: nothing to offload")
    if m < 1:
        raise ValueError("population must be positive")
    population = []
    for _ in range(m):
        population.append(tuple(rng.randint(0, 1) for _ in range(gene_len)))
    return population


def roulette_pick(population: list, rng: random.Random) -> Individual:
    """Fitness-proportional draw (fitness > 0 always)."""
    edges = []
    acc = 0.0
    for ind in population:
        acc += ind.fitness
        edges.append(acc)
    return population[bisect.bisect_left(edges, rng.random() * acc)]


def crossover(parent_a: Genome, parent_b: Genome, pc: float, rng: random.Random) -> tuple:
    if len(parent_a) != len(parent_b):
        raise LengthMismatch(f"{len(parent_a)} vs {len(parent_b)}")
    n = len(parent_a)
    if n < 2 or rng.random() >= pc:
        return tuple(parent_a), tuple(parent_b)
    cut = rng.randint(1, n - 1)
    return tuple(parent_a[:cut]) + tuple(parent_b[cut:]), tuple(parent_b[:cut]) + tuple(parent_a[cut:])


def mutate(genome: Genome, pm: float, rng: random.Random) -> Genome:
    return tuple((bit ^ 1) if rng.random() < pm else bit for bit in genome)


class EvalCache:
    """Genome -> (effective time, timed_out, penalized, diagnostic)."""

    def __init__(self):
        self._store: dict = {}

    def __contains__(self, genome) -> bool:
        return genome in self._store

    def get(self, genome):
        return self._store[genome]

    def put(self, genome, value) -> None:
        self._store[genome] = value

    def __len__(self) -> int:
        return len(self._store)


def _effective(measured, penalty_time_s: float) -> tuple:
    """Failure -> penalty ("penalty"); timeout -> penalty but "fresh" (ga.py:164-169)."""
    if measured.failure is not None:
        return penalty_time_s, False, True, measured.failure
    if measured.timed_out:
        return penalty_time_s, True, False, ""
    return measured.seconds, False, False, ""


def _individual(genome, value, cached: bool) -> Individual:
    time_s, timed_out, penalized, diag = value
    source = "cache" if cached else ("penalty" if penalized else "fresh")
    return Individual(genome, time_s, fitness(time_s), source, timed_out, diag)


def evaluate_with_cache(genome, evaluator, cache: EvalCache, penalty_time_s: float) -> Individual:
    if genome in cache:
        return _individual(genome, cache.get(genome), True)
    value = _effective(evaluator.measure(genome), penalty_time_s)
    cache.put(genome, value)
    return _individual(genome, value, False)


@dataclass
class GAResult:
    best: Individual
    records: list
    evaluations: int

    @property
    def best_time_s(self) -> float:
        return self.best.time_s


def _measure_all(evaluator, pending: list) -> dict:
    width = getattr(evaluator, "max_concurrency", 1) or 1
    if width > 1 and len(pending) > 1:
        with ThreadPoolExecutor(max_workers=width) as pool:
            return dict(zip(pending, pool.map(evaluator.measure, pending)))
    return {g: evaluator.measure(g) for g in pending}


def _evaluate_generation(genomes: list, evaluator, cache: EvalCache, config: GAConfig) -> tuple:
    pending = list(dict.fromkeys(g for g in genomes if g not in cache))
    measured = _measure_all(evaluator, pending)
    out = []
    for g in genomes:
        if g in cache:
            out.append(_individual(g, cache.get(g), True))
        else:
            value = _effective(measured[g], config.penalty_time_s)
            cache.put(g, value)
            out.append(_individual(g, value, False))
    return out, len(pending)


def _next_generation(individuals: list, config: GAConfig, rng: random.Random) -> list:
    order = sorted(range(len(individuals)), key=lambda i: (-individuals[i].fitness, i))
    nxt = [individuals[i].genome for i in order[:config.elitism_count]]
    while len(nxt) < config.population:
        if config.population - len(nxt) == 1:
            lone = roulette_pick(individuals, rng)
            nxt.append(mutate(lone.genome, config.mutation_rate, rng))
            break
        a = roulette_pick(individuals, rng)
        b = roulette_pick(individuals, rng)
        ca, cb = crossover(a.genome, b.genome, config.crossover_rate, rng)
        nxt.append(mutate(ca, config.mutation_rate, rng))
        nxt.append(mutate(cb, config.mutation_rate, rng))
    return nxt


def run_ga(config: GAConfig, gene_len: int, evaluator,
           on_generation: Optional[Callable] = None) -> GAResult:
    """T generations of evaluate -> select (+elite) -> crossover -> mutate; best-ever wins."""
    rng = random.Random(config.rng_seed)
    genomes = init_population(gene_len, config.population, rng)
    cache = EvalCache()
    records = []
    best: Optional[Individual] = None
    fresh_total = 0
    for gen in range(config.generations):
        individuals, fresh = _evaluate_generation(genomes, evaluator, cache, config)
        fresh_total += fresh
        for ind in individuals:
            if best is None or ind.time_s < best.time_s:
                best = ind
        rec = GenerationRecord(gen, individuals, best.genome, best.time_s)
        records.append(rec)
        if on_generation is not None:
            on_generation(rec)
        if gen + 1 < config.generations:
            genomes = _next_generation(individuals, config, rng)
    return GAResult(best, records, fresh_total)
