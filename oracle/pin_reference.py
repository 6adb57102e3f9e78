"""Pin the oracle and the host logic to the REFERENCE itself (dev container only).

Runs the reference package from /root/reference/pkg/src (read-only, imported,
never copied) and writes golden fixtures under tests/golden/ that the test
suite checks on any machine (the GPU box has no /root/reference):

* himeno_<size>_n<nn>.stdout -- stdout of the reference's own
  ExternalEvaluator.run_for_output (acctuner/evaluators.py:183-188) on the
  Himeno C-subset text, with the reference template "gcc -O2 -w {src} -o {bin}"
  (pragmas ignored: SURVEY.md §8(c)).  Also the stdout of the reference's
  emitted OpenACC variant (emit_variant, emitter.py:132) for a few genomes,
  which must be identical (the pragmas are ignored by gcc).
* plans_himeno.json.gz -- Planner.plan and Planner.plan_transfers
  (transfer.py:184-193, 413-418) for all 2^13 genomes.
* ft_<class>.stdout -- the same for the NAS FT restatement (apps/ft.py) with the
  template "gcc -O2 -w {src} -o {bin} -lm"; its checksums equal NPB's published
  verification values (tests/test_ft.py).
* plans_ft_s.json.gz -- Planner.plan / plan_transfers for FT class S on all 36
  single-gene genomes, the all-ones genome and 400 seeded random genomes.
* ga_streams.json -- run_ga (ga.py:183-211) GenerationRecord streams for
  several configs under a deterministic replay evaluator (fixed time table,
  including failures and timeouts).

    PYTHONPATH=/root/reference/pkg/src python oracle/pin_reference.py
"""

from __future__ import annotations

import gzip
import hashlib
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, "/root/reference/pkg/src")

from acctuner.classify import StaticRuleProbe, classify_project, eligible_ids  # noqa: E402
from acctuner.code_model import analyze_project  # noqa: E402
from acctuner.emitter import emit_variant  # noqa: E402
from acctuner.evaluators import CommandConfig, ExternalEvaluator, MeasuredTime  # noqa: E402
from acctuner.ga import GAConfig, run_ga  # noqa: E402
from acctuner.transfer import Planner  # noqa: E402

from paper_2002_12115_b200.apps import ft, himeno  # noqa: E402

GOLDEN = ROOT / "tests" / "golden"
CASES = [("XXS", 1), ("XXS", 3), ("XS", 3), ("XS", 1), ("S", 2), ("M", 2)]
VARIANT_GENOMES = ["0000000100100", "1001001000000", "0010010010010"]


def _project(size_name, nn):
    sz = himeno.size(size_name)
    fid = himeno.source_file_id(sz)
    text = himeno.source_text(sz, nn)
    proj = analyze_project([(fid, text)])
    verdicts = classify_project(proj, StaticRuleProbe())
    return fid, text, proj, verdicts


def pin_stdout():
    ev = ExternalEvaluator(CommandConfig("gcc -O2 -w -mcmodel=medium {src} -o {bin}", "{bin}",
                                         600.0, 1), build_variant=None)
    for size_name, nn in CASES:
        fid, text, proj, verdicts = _project(size_name, nn)
        out = ev.run_for_output({fid: text})
        (GOLDEN / f"himeno_{size_name.lower()}_n{nn}.stdout").write_text(out)
        print(f"{size_name} n={nn}: {out.split()}")
        if size_name == "XS" and nn == 3:
            planner = Planner(proj.loops, proj.refs, eligible_ids(verdicts))
            for g in VARIANT_GENOMES:
                genome = tuple(int(c) for c in g)
                variant = emit_variant(proj, genome, verdicts, planner.plan(genome))
                vout = ev.run_for_output(variant.texts)
                if vout != out:
                    raise SystemExit(f"emitted variant {g} changed the output")
                (GOLDEN / f"himeno_xs_n3_variant_{g}.c").write_text(variant.texts[fid])


def _sig(e):
    return [e.var, e.direction.value, list(e.members), e.open_file, list(e.open_span),
            e.close_file, list(e.close_span), list(e.present_sites), e.temp_region]


def pin_plans():
    fid, text, proj, verdicts = _project("XS", 3)
    elig = eligible_ids(verdicts)
    planner = Planner(proj.loops, proj.refs, elig)
    n = len(elig)
    doc = {"file": fid, "eligible": elig, "plans": {}, "raw": {}}
    for value in range(1 << n):
        g = tuple((value >> (n - 1 - i)) & 1 for i in range(n))
        key = "".join(map(str, g))
        doc["plans"][key] = [_sig(e) for e in planner.plan(g).entries]
        doc["raw"][key] = [_sig(e) for e in planner.plan_transfers(g).entries]
    with gzip.open(GOLDEN / "plans_himeno.json.gz", "wt") as fh:
        json.dump(doc, fh, separators=(",", ":"), sort_keys=True)
    print(f"plans: {len(doc['plans'])} genomes")


def replay_time(genome) -> MeasuredTime:
    """Deterministic fake measurement: hash -> time; some failures / timeouts."""
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

    def measure(self, genome):
        return replay_time(genome)


GA_CONFIGS = [
    dict(population=4, generations=4, rng_seed=0),
    dict(population=10, generations=10, rng_seed=1),
    dict(population=20, generations=20, rng_seed=2),
    dict(population=7, generations=6, rng_seed=3, elitism_count=2),
    dict(population=10, generations=10, rng_seed=4, crossover_rate=0.0, mutation_rate=0.3),
    dict(population=30, generations=20, rng_seed=5),
]


def pin_ga():
    streams = []
    for cfg_doc in GA_CONFIGS:
        for gene_len in (13, 65):
            res = run_ga(GAConfig(**cfg_doc), gene_len, Replay(8))
            streams.append({"config": cfg_doc, "gene_len": gene_len,
                            "evaluations": res.evaluations,
                            "best": res.best.to_json(),
                            "records": [r.to_json() for r in res.records]})
    (GOLDEN / "ga_streams.json").write_text(json.dumps(streams, sort_keys=True) + "\n")
    print(f"ga: {len(streams)} streams")


FT_SAMPLES = 400


def ft_genomes(n: int) -> list:
    import random
    rng = random.Random(2002_12115)
    out = [tuple(int(i == j) for j in range(n)) for i in range(n)]
    out.append((1,) * n)
    out += [tuple(rng.randint(0, 1) for _ in range(n)) for _ in range(FT_SAMPLES)]
    return out


def pin_ft():
    ev = ExternalEvaluator(CommandConfig("gcc -O2 -w {src} -o {bin} -lm", "{bin}", 600.0, 1),
                           build_variant=None)
    for name in ("S", "W", "A"):
        c = ft.ft_class(name)
        fid, text = ft.source_file_id(c), ft.source_text(c)
        out = ev.run_for_output({fid: text})
        (GOLDEN / f"ft_{name.lower()}.stdout").write_text(out)
        print(f"FT {name}: {out.split()[:2]} ...")
    c = ft.ft_class("S")
    proj = analyze_project([(ft.source_file_id(c), ft.source_text(c))])
    elig = eligible_ids(classify_project(proj, StaticRuleProbe()))
    planner = Planner(proj.loops, proj.refs, elig)
    doc = {"file": ft.source_file_id(c), "eligible": elig, "plans": {}, "raw": {}}
    for g in ft_genomes(len(elig)):
        key = "".join(map(str, g))
        doc["plans"][key] = [_sig(e) for e in planner.plan(g).entries]
        doc["raw"][key] = [_sig(e) for e in planner.plan_transfers(g).entries]
    with gzip.open(GOLDEN / "plans_ft_s.json.gz", "wt") as fh:
        json.dump(doc, fh, separators=(",", ":"), sort_keys=True)
    print(f"ft plans: {len(doc['plans'])} genomes")


def main():
    GOLDEN.mkdir(parents=True, exist_ok=True)
    if "--ft" in sys.argv:
        pin_ft()
        return
    pin_stdout()
    pin_plans()
    pin_ga()
    pin_ft()


if __name__ == "__main__":
    main()
