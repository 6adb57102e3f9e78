"""Planner parity: plan.Planner == reference acctuner.transfer.Planner.

Against committed goldens (all 2^13 genomes, batched and raw plans) on any
machine, and against the live reference when it is mounted.
"""
import gzip
import json

import pytest

from conftest import GOLDEN
from paper_2002_12115_b200.apps import himeno
from paper_2002_12115_b200.plan import Direction, Planner


def _sig(e):
    return [e.var, e.direction.value, list(e.members), e.open_file, list(e.open_span),
            e.close_file, list(e.close_span), list(e.present_sites), e.temp_region]


@pytest.fixture(scope="module")
def golden():
    with gzip.open(GOLDEN / "plans_himeno.json.gz", "rt") as fh:
        return json.load(fh)


@pytest.fixture(scope="module")
def planner():
    prog = himeno.program()
    return Planner(prog.model.loops, prog.model.refs, list(prog.eligible))


def test_all_genomes_batched_and_raw(golden, planner):
    assert len(golden["plans"]) == 8192
    bad = []
    for key, want in golden["plans"].items():
        g = tuple(int(c) for c in key)
        if [_sig(e) for e in planner.plan(g).entries] != want:
            bad.append(("plan", key))
        if [_sig(e) for e in planner.plan_transfers(g).entries] != golden["raw"][key]:
            bad.append(("raw", key))
    assert not bad, bad[:5]


def test_known_plans(planner):
    # batched plan of 0000000100100 opens the arrays once at loop 6
    plan = planner.plan((0, 0, 0, 0, 0, 0, 0, 1, 0, 0, 1, 0, 0))
    by_var = {e.var: e for e in plan.entries}
    assert by_var["p"].direction is Direction.COPY and by_var["p"].open_loop == 6
    assert by_var["jacobi:gosa"].open_loop == 7 and not by_var["jacobi:gosa"].temp_region
    assert all(by_var[v].temp_region for v in ("p", "a", "b", "c", "wrk1", "bnd", "omega"))
    raw = planner.plan_transfers((0, 0, 0, 0, 0, 0, 0, 1, 0, 0, 1, 0, 0))
    assert {e.open_loop for e in raw.entries if e.var == "p"} == {7, 10}
    assert raw.total_events() > plan.total_events() - 1


def test_all_cpu_genome_has_empty_plan(planner):
    assert planner.plan((0,) * 13).entries == []


def test_live_reference_spot_check(reference, planner):
    from acctuner.code_model import analyze_project
    from acctuner.classify import StaticRuleProbe, classify_project, eligible_ids
    from acctuner.transfer import Planner as RefPlanner
    sz = himeno.size("M")
    proj = analyze_project([(himeno.source_file_id(sz), himeno.source_text(sz, 5))])
    elig = eligible_ids(classify_project(proj, StaticRuleProbe()))
    ref = RefPlanner(proj.loops, proj.refs, elig)
    mine = Planner(proj.loops, proj.refs, elig)   # duck-typed on the reference model
    for value in range(0, 8192, 37):
        g = tuple((value >> (12 - i)) & 1 for i in range(13))
        assert [_sig(e) for e in mine.plan(g).entries] == [_sig(e) for e in ref.plan(g).entries]
        assert ([_sig(e) for e in mine.plan_transfers(g).entries]
                == [_sig(e) for e in ref.plan_transfers(g).entries])
