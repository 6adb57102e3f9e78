"""Schedule lowering: genome + kinds + plan -> native events (no GPU needed)."""
import pytest

from paper_2002_12115_b200 import native as N
from paper_2002_12115_b200.apps import himeno
from paper_2002_12115_b200.errors import PlanInconsistent
from paper_2002_12115_b200.evaluator import valid_genomes
from paper_2002_12115_b200.lower import loop_kinds, lower, plan_events
from paper_2002_12115_b200.plan import Planner

PROG = himeno.program()
LOOPS, REFS = PROG.model.loops, PROG.model.refs
ELIG = list(PROG.eligible)
PLANNER = Planner(LOOPS, REFS, ELIG)


def g(s):
    return tuple(int(c) for c in s)


def test_valid_genome_count():
    assert len(valid_genomes(LOOPS, ELIG)) == 272


def test_nested_rejected_and_outermost():
    genome = g("0000001100000")
    gene = dict(zip(ELIG, genome))
    kinds, why = loop_kinds(LOOPS, gene, PROG.kinds, "reject")
    assert kinds is None and "nested compute construct" in why
    kinds, why = loop_kinds(LOOPS, gene, PROG.kinds, "outermost")
    assert why is None
    assert kinds[6] == N.K_PARALLEL_LOOP and kinds[7] == N.K_COVERED and kinds[12] == N.K_COVERED
    low = lower(genome, ELIG, PROG.kinds, LOOPS, REFS, PLANNER.plan(genome), 3, 0,
                nested_policy="outermost")
    assert low.failure is None


def test_kinds_follow_classifier():
    kinds, _ = loop_kinds(LOOPS, dict(zip(ELIG, g("1001001000000"))), PROG.kinds)
    assert kinds[0] == N.K_KERNELS and kinds[3] == N.K_KERNELS
    assert kinds[6] == N.K_PARALLEL_LOOP
    assert kinds[1] == N.K_COVERED and kinds[7] == N.K_COVERED and kinds[9] == N.K_COVERED
    kinds, _ = loop_kinds(LOOPS, dict(zip(ELIG, g("0010010010010"))), PROG.kinds)
    assert kinds[2] == N.K_PARALLEL_LOOP and kinds[8] == N.K_KERNELS and kinds[7] == N.K_HOST


@pytest.mark.parametrize("mode", ["batched", "raw"])
def test_events_realise_every_plan_entry(mode):
    for genome in valid_genomes(LOOPS, ELIG):
        plan = PLANNER.plan(genome) if mode == "batched" else PLANNER.plan_transfers(genome)
        gene = dict(zip(ELIG, genome))
        events = plan_events(plan, LOOPS, REFS, gene)
        for idx, e in enumerate(plan.entries):
            mine = [ev for ev in events if ev[5] == idx]
            ops = sorted(ev[2] for ev in mine)
            if e.temp_region:
                want = ([N.EV_UPDATE_DEVICE] if e.direction.into_device else []) + \
                       ([N.EV_UPDATE_SELF] if e.direction.out_of_device else [])
                got = [o for o in ops if o in (N.EV_UPDATE_DEVICE, N.EV_UPDATE_SELF)]
                assert got == sorted(want)
            else:
                enter = [ev for ev in mine if ev[2] == N.EV_DATA_ENTER]
                leave = [ev for ev in mine if ev[2] == N.EV_DATA_EXIT]
                assert len(enter) == 1 and len(leave) == 1
                assert enter[0][4] == int(e.direction.into_device)
                assert leave[0][4] == int(e.direction.out_of_device)
                assert enter[0][0] == e.open_loop and leave[0][0] == e.close_loop
            assert len([ev for ev in mine if ev[2] == N.EV_PRESENT]) == len(e.present_sites)
        declared = {ev[3] for ev in events if ev[2] == N.EV_DECLARE}
        assert declared == {N.VAR_ID[e.var] for e in plan.entries if e.temp_region}


def test_inconsistent_plan_rejected():
    plan = PLANNER.plan(g("0000000100100"))
    with pytest.raises(PlanInconsistent):
        plan_events(plan, LOOPS, REFS, dict(zip(ELIG, g("0000000000000"))))


def test_schedule_struct():
    genome = g("0000000100100")
    low = lower(genome, ELIG, PROG.kinds, LOOPS, REFS, PLANNER.plan(genome), 7,
                N.FLAG_COHERENCE_GUARD, 12.5)
    s = low.schedule
    assert s.n_loops == 13 and s.nn == 7 and s.timeout_s == 12.5
    assert list(s.loop_kind) == [0, 0, 0, 0, 0, 0, 0, 1, 4, 4, 1, 4, 4]
    assert s.n_events == len(low.events)
    assert [s.events[i].op for i in range(s.n_events)] == [ev[2] for ev in low.events]
