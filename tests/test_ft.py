"""NAS FT restatement (apps/ft.py): pinned to NPB's verification checksums and to the
reference's own front-end and planner.

* the reference's ExternalEvaluator stdout (gcc -O2, pragmas ignored; committed by
  oracle/pin_reference.py) reproduces NPB FT's published class S / W / A checksums to NPB's
  1e-12 relative tolerance -- the restatement is the NPB algorithm;
* the committed program model is the reference's analyze_project + StaticRuleProbe
  output (93 loops, 79 genes);
* plan.Planner equals the reference Planner on 480 FT genomes (golden).
"""
import gzip
import json

import pytest

from conftest import GOLDEN
from paper_2002_12115_b200.apps import ft
from paper_2002_12115_b200.plan import Planner


def _sig(e):
    return [e.var, e.direction.value, list(e.members), e.open_file, list(e.open_span),
            e.close_file, list(e.close_span), list(e.present_sites), e.temp_region]


@pytest.mark.parametrize("cls", ["S", "W", "A"])
def test_reference_stdout_matches_npb_checksums(cls):
    out = (GOLDEN / f"ft_{cls.lower()}.stdout").read_text()
    assert ft.checksum_error(out, cls) <= ft.VERIFY_RTOL


def test_program_model_shape():
    prog = ft.program("S")
    assert len(prog.model.loops) == 93
    assert prog.gene_length == 79
    kinds = {lid: k.value for lid, k in prog.kinds.items()}
    assert kinds[0] == "kernels" and kinds[2] == "parallel loop" and kinds[91] == "kernels"
    # the FFT's k loops (butterfly offsets i*lk + k) are rejected by the static probe;
    # the printf loop has a call
    assert 14 not in prog.eligible and 92 not in prog.eligible


def test_planner_matches_reference_golden():
    with gzip.open(GOLDEN / "plans_ft_s.json.gz", "rt") as fh:
        golden = json.load(fh)
    prog = ft.program("S")
    assert golden["eligible"] == list(prog.eligible)
    planner = Planner(prog.model.loops, prog.model.refs, list(prog.eligible))
    bad = []
    for key, want in golden["plans"].items():
        g = tuple(int(c) for c in key)
        if [_sig(e) for e in planner.plan(g).entries] != want:
            bad.append(("plan", key))
        if [_sig(e) for e in planner.plan_transfers(g).entries] != golden["raw"][key]:
            bad.append(("raw", key))
    assert len(golden["plans"]) == 480 and not bad, bad[:3]


def test_gcc_build_of_the_text_verifies(tmp_path):
    """The program text compiled the way the reference's template does verifies (class S)."""
    import shutil
    import subprocess
    if not shutil.which("gcc"):
        pytest.skip("gcc unavailable")
    c = ft.ft_class("S")
    src = tmp_path / ft.source_file_id(c)
    src.write_text(ft.source_text(c))
    subprocess.run(["gcc", "-O2", "-w", str(src), "-o", str(tmp_path / "ft"), "-lm"], check=True)
    out = subprocess.run([str(tmp_path / "ft")], capture_output=True, text=True, check=True).stdout
    assert ft.checksum_error(out, "S") <= ft.VERIFY_RTOL
