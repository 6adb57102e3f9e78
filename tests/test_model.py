"""Program model: committed structural JSON loads to the reference's model."""
from paper_2002_12115_b200.apps import himeno
from paper_2002_12115_b200.model import dump_structural, load_structural


def test_loop_tree():
    prog = himeno.program()
    loops = prog.model.loops
    assert len(loops) == 13 and prog.gene_length == 13
    parents = {l.loop_id: l.parent_loop for l in loops}
    assert parents == {0: None, 1: 0, 2: 1, 3: None, 4: 3, 5: 4, 6: None, 7: 6, 8: 7, 9: 8,
                       10: 6, 11: 10, 12: 11}
    shapes = [l.shape for l in loops]
    assert shapes[6] == "non_tight" and shapes[7] == "tight_outer" and shapes[9] == "tight_inner"
    kinds = [prog.kinds[i].value for i in range(13)]
    assert kinds == ["kernels", "kernels", "parallel loop", "kernels", "kernels", "parallel loop",
                     "parallel loop", "kernels", "kernels", "parallel loop", "kernels", "kernels",
                     "parallel loop"]


def test_region_sequence_and_index_vars():
    refs = himeno.program().model.refs
    assert refs.region_sequence == ["pre", 0, 1, 2, "host:1", 3, 4, 5, "host:2", 6, 7, 8, 9,
                                    10, 11, 12, "post"]
    keys = {v.key for v in refs.plannable()}
    assert "jacobi:i" not in keys and "initmt:k" not in keys and "jacobi:n" not in keys
    assert {"p", "a", "b", "c", "wrk2", "jacobi:gosa", "jacobi:nn"} <= keys


def test_dump_load_roundtrip():
    model = himeno.program().model
    doc = dump_structural(model)
    again = load_structural(doc)
    assert dump_structural(again) == doc


def test_matches_reference_front_end(reference):
    from acctuner.code_model import analyze_project
    from acctuner.code_model import dump_structural as ref_dump
    sz = himeno.size("XS")
    proj = analyze_project([(himeno.source_file_id(sz), himeno.source_text(sz, 3))])
    want = ref_dump(proj)
    mine = dump_structural(himeno.program().model, include_index_keys=False)
    assert mine == want
    assert sorted(proj.refs.index_var_keys) == sorted(himeno.program().model.refs.index_var_keys)
