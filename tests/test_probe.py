"""B200 probe: same classification as the static probe on Himeno, through the
reference's own classify_loop (duck-typed probe interface)."""
import pytest

from paper_2002_12115_b200.apps import himeno
from paper_2002_12115_b200.model import LoopInfo
from paper_2002_12115_b200.probe import B200Probe


def test_accepts_every_himeno_loop_and_kind():
    prog = himeno.program()
    probe = B200Probe()
    for l in prog.model.loops:
        for kind in ("kernels", "parallel loop", "parallel loop vector"):
            assert probe.probe(l, kind).accepted
    assert "sequential" in probe.probe(prog.model.loops.get(6), "parallel loop").diagnostic


def test_rejects_unknown_loops():
    probe = B200Probe()
    stranger = LoopInfo(99, "x.c", (0, 1), 0, None, "i", None, "single")
    assert not probe.probe(stranger, "kernels").accepted
    moved = LoopInfo(7, "x.c", (0, 1), 0, None, "i", None, "single")   # wrong parent/shape
    assert not probe.probe(moved, "kernels").accepted


def test_reference_classify_with_b200_probe(reference):
    from acctuner.classify import StaticRuleProbe, classify_project, eligible_ids, kind_map
    from acctuner.code_model import analyze_project
    sz = himeno.size("XS")
    proj = analyze_project([(himeno.source_file_id(sz), himeno.source_text(sz, 3))])
    mine = classify_project(proj, B200Probe())
    static = classify_project(proj, StaticRuleProbe())
    assert eligible_ids(mine) == eligible_ids(static) == list(range(13))
    assert kind_map(mine) == kind_map(static)


@pytest.mark.gpu
def test_execution_probe_runs_every_loop_and_kind(gpu):
    """execute=True: every (loop, kind) of the Himeno program is run as its one-gene
    pattern on XS (NaN-poisoned device memory) and reproduces the all-CPU program."""
    prog = himeno.program()
    probe = B200Probe(execute=True, size="XS", nn=2)
    try:
        for l in prog.model.loops:
            for kind in ("kernels", "parallel loop", "parallel loop vector"):
                r = probe.probe(l, kind)
                assert r.accepted, (l.loop_id, kind, r.diagnostic)
                assert "bit-exact" in r.diagnostic
        # cached: a second call does not run again
        again = probe.probe(prog.model.loops.get(9), "kernels")
        assert again.accepted
    finally:
        probe.close()


@pytest.mark.gpu
def test_reference_classify_with_executing_probe(gpu, reference):
    """The reference's classify_project with the executing probe: the same genes and
    kinds as its static probe, each backed by a verified run."""
    from acctuner.classify import StaticRuleProbe, classify_project, eligible_ids, kind_map
    from acctuner.code_model import analyze_project
    sz = himeno.size("XS")
    proj = analyze_project([(himeno.source_file_id(sz), himeno.source_text(sz, 3))])
    probe = B200Probe(execute=True, size="XS", nn=2)
    try:
        mine = classify_project(proj, probe)
    finally:
        probe.close()
    static = classify_project(proj, StaticRuleProbe())
    assert eligible_ids(mine) == eligible_ids(static) == list(range(13))
    assert kind_map(mine) == kind_map(static)
