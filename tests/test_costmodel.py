"""Cost-model evaluator: parity with the reference API and calibration recovery."""
import json
import random

import pytest

from paper_2002_12115_b200 import costmodel as cm
from paper_2002_12115_b200 import ga
from paper_2002_12115_b200.apps import himeno
from paper_2002_12115_b200.errors import EnumerationTooLarge, ModelIncomplete
from paper_2002_12115_b200.evaluator import valid_genomes

PROG = himeno.program()
LOOPS, REFS, ELIG = PROG.model.loops, PROG.model.refs, list(PROG.eligible)


def synthetic_model(seed=0):
    rng = random.Random(seed)
    return cm.CostModel(
        overhead_s=0.01,
        loop_cpu_s={l: rng.uniform(0.0, 0.2) for l in ELIG},
        loop_gpu_s={l: rng.uniform(0.0, 0.02) for l in ELIG},
        var_bytes=cm.var_bytes_of(REFS), bandwidth_bytes_per_s=2.5e10, latency_s=1e-5)


def test_json_roundtrip_and_validation():
    m = synthetic_model()
    again = cm.CostModel.from_json(json.loads(json.dumps(m.to_json())))
    assert again.to_json() == m.to_json()
    with pytest.raises(ValueError):
        cm.CostModel(0, {}, {}, {}, 0.0, 0.0)
    with pytest.raises(ModelIncomplete):
        m.transfer_event_s("nope")


def test_all_zero_genome_is_cpu_sum():
    m = synthetic_model()
    ev = cm.CostModelEvaluator(m, LOOPS, REFS, ELIG)
    t = ev.measure((0,) * 13).seconds
    assert abs(t - (m.overhead_s + sum(m.loop_cpu_s.values()))) < 1e-15


def test_brute_force_optimum_dominates_ga():
    m = synthetic_model(3)
    best, t = cm.brute_force_optimum(m, LOOPS, REFS, ELIG)
    ev = cm.CostModelEvaluator(m, LOOPS, REFS, ELIG)
    res = ga.run_ga(ga.GAConfig(population=10, generations=10, rng_seed=1), 13, ev)
    assert t <= res.best_time_s + 1e-15
    with pytest.raises(EnumerationTooLarge):
        cm.brute_force_optimum(m, LOOPS, REFS, list(range(21)))


def test_matches_reference_costmodel(reference):
    from acctuner.code_model import analyze_project
    from acctuner.classify import StaticRuleProbe, classify_project, eligible_ids
    from acctuner.evaluators import CostModel as RefModel, evaluate_costmodel as ref_eval
    from acctuner.transfer import Planner as RefPlanner
    sz = himeno.size("XS")
    proj = analyze_project([(himeno.source_file_id(sz), himeno.source_text(sz, 3))])
    elig = eligible_ids(classify_project(proj, StaticRuleProbe()))
    m = synthetic_model(5)
    rm = RefModel.from_json(m.to_json())
    rp = RefPlanner(proj.loops, proj.refs, elig)
    for value in range(0, 8192, 61):
        g = tuple((value >> (12 - i)) & 1 for i in range(13))
        want = ref_eval(g, rp.plan(g), rm, elig, proj.refs)
        got = cm.evaluate_costmodel(g, rp.plan(g), m, elig, proj.refs)
        assert got == want


def test_calibration_recovers_an_additive_model():
    truth = synthetic_model(7)
    ev = cm.CostModelEvaluator(truth, LOOPS, REFS, ELIG)
    genomes = valid_genomes(LOOPS, ELIG)
    samples = [(g, ev.measure(g).seconds) for g in genomes]
    cal = cm.calibrate(samples, LOOPS, REFS, ELIG, truth.bandwidth_bytes_per_s, truth.latency_s)
    assert cal.residual_rms_s < 1e-6
    pred = [cm.CostModelEvaluator(cal.model, LOOPS, REFS, ELIG).measure(g).seconds
            for g in genomes]
    assert cm.spearman(pred, [s for _, s in samples]) > 0.999
    assert cm.optimum_over(cal.model, LOOPS, REFS, ELIG, genomes)[0] == \
        cm.optimum_over(truth, LOOPS, REFS, ELIG, genomes)[0]


def test_nest_aware_modes_and_recovery():
    modes = cm.loop_modes((0, 0, 0, 0, 0, 0, 1, 0, 0, 0, 0, 0, 0), LOOPS, ELIG)
    assert modes[6] == "gpu" and all(modes[l] == "covered" for l in range(7, 13))
    assert modes[0] == "cpu" and modes[1] == "inside"
    modes = cm.loop_modes((0, 0, 0, 0, 0, 0, 0, 0, 1, 0, 0, 0, 0), LOOPS, ELIG)
    assert modes[6] == "driver" and modes[7] == "driver" and modes[8] == "gpu"
    assert modes[10] == "cpu" and modes[9] == "covered"
    truth = synthetic_model(11)
    ev = cm.CostModelEvaluator(truth, LOOPS, REFS, ELIG, nest_aware=True)
    genomes = valid_genomes(LOOPS, ELIG)
    samples = [(g, ev.measure(g).seconds) for g in genomes]
    cal = cm.calibrate(samples, LOOPS, REFS, ELIG, truth.bandwidth_bytes_per_s,
                       truth.latency_s, nest_aware=True)
    assert cal.residual_rms_s < 1e-6
    assert cm.optimum_over(cal.model, LOOPS, REFS, ELIG, genomes, nest_aware=True)[0] == \
        cm.optimum_over(truth, LOOPS, REFS, ELIG, genomes, nest_aware=True)[0]
