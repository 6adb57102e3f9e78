"""Generated executors (codegen.py + csrc/gen_runtime.cuh + generic.py).

CPU: the generator parses the program texts, the libraries export the ABI and carry the
model's loop / variable tables, and a host-only context runs the all-CPU pattern to the
reference's own stdout byte for byte (FT S / W, Himeno XS).  GPU: FT patterns whose
device semantics are exact (no false accepts of the static probe) reproduce NPB's
checksums; every single-gene pattern runs without a device fault; the generated Himeno
executor agrees with the hand-written library; run_ga drives the FT evaluator.
"""
import random

import pytest

from conftest import GOLDEN
from paper_2002_12115_b200 import codegen, generic
from paper_2002_12115_b200.apps import ft, himeno

GOLD = {"ft_s": "ft_s.stdout", "ft_w": "ft_w.stdout", "ft_a": "ft_a.stdout",
        "himeno_xs": "himeno_xs_n3.stdout"}


def test_codegen_parses_the_programs():
    p = codegen.CProgram(ft.source_text("S"))
    assert [f.name for f in p.funcs] == ["main"]
    assert p.gmap["u0r"].dims == [64, 64, 64] and p.gmap["seeds"].dims == [64]
    h = codegen.CProgram(himeno.source_text(himeno.size("XS"), 3))
    assert h.gmap["a"].dims == [4, 33, 33, 65]
    jac = next(f for f in h.funcs if f.name == "jacobi")
    assert {d.name for d in jac.locals} >= {"gosa", "s0", "ss"}


def test_kernel_plans_follow_the_directive_semantics():
    prog = ft.program("S")
    p = codegen.CProgram(ft.source_text("S"))
    loops = prog.model.loops
    kp = codegen.plan_kernel(p, loops.get(0), "kernels", loops)
    assert kp.mode == "grid" and len(kp.levels) == 3          # tight 3-D nest collapsed
    kp = codegen.plan_kernel(p, loops.get(5), "kernels", loops)
    assert kp.mode == "seq" and [d.name for d in kp.carried] == ["x"]
    kp = codegen.plan_kernel(p, loops.get(3), "kernels", loops)        # seed chain
    assert kp.mode == "seq" and "rx" in [d.name for d in kp.carried]
    kp = codegen.plan_kernel(p, loops.get(91), "kernels", loops)
    assert [d.name for d in kp.reductions] == ["cr", "ci"]
    kp = codegen.plan_kernel(p, loops.get(4), "parallel loop", loops)
    assert kp.mode == "grid" and "x" in [d.name for d in kp.privates] and not kp.carried
    # the FFT butterfly loop i (parallel loop): one gang per i; its k x j nest is the
    # vector region, spread over several blocks (nothing it writes is read in the gang)
    kinds = {k: v.value for k, v in prog.kinds.items()}
    kp = codegen.plan_kernel(p, loops.get(13), "parallel loop", loops, kinds)
    assert kp.mode == "gang" and kp.vsplit
    assert [(r.loop_id, [h.var for h in hs]) for r, hs in kp.vec] == [(14, ["k", "j"])]
    # the line-batch loop a: its copy / stage loops need barriers between them
    kp = codegen.plan_kernel(p, loops.get(9), "parallel loop", loops, kinds)
    assert kp.mode == "gang" and not kp.vsplit and len(kp.vec) >= 3


@pytest.mark.parametrize("app", generic.APPS)
def test_library_tables(app):
    lib = generic.load(app)
    prog = generic.app_specs()[app].program()
    assert lib.n_loops == len(prog.model.loops)
    for lid in prog.eligible:
        assert lib.lib.hpg_loop_kind(lid) > 0, lid
    ev_keys = {e.var for g in [(1,) * len(prog.eligible)] for e in
               generic.Planner(prog.model.loops, prog.model.refs, list(prog.eligible))
               .plan(g).entries}
    assert ev_keys <= set(lib.var_id), ev_keys - set(lib.var_id)


@pytest.mark.parametrize("app", generic.APPS)
def test_host_only_all_cpu_pattern_matches_reference_stdout(app):
    with generic.GenEvaluator(app, devices=[-1]) as ev:
        g = (0,) * ev.gene_length
        m = ev.measure(g)
        assert m.seconds is not None, m
        assert ev.outputs[g] == (GOLDEN / GOLD[app]).read_text()
        # a device pattern on a host-only context fails cleanly (no crash)
        m1 = ev.measure((1,) + (0,) * (ev.gene_length - 1))
        assert m1.failure and "no CUDA device" in m1.failure


def test_random_ft_genomes_lower():
    with generic.GenEvaluator("ft_s", devices=[-1]) as ev:
        rng = random.Random(5)
        for _ in range(50):
            g = tuple(rng.randint(0, 1) for _ in range(ev.gene_length))
            low = ev.lowered(g)
            assert low.failure is not None or low.schedule.n_loops == 93


# ---------------------------------------------------------------------------- GPU

# FT loops whose device versions are exact under their directive kind: the twiddle,
# seed (sequential device thread) and plane-fill loops, every copy / butterfly / evolve
# / checksum loop.  The static probe also accepts the scalar-carried i loop (6), the
# roots loop (7), the FFT stage loops (12, 24, ...), the line-batch loops (9, 21, ...)
# and the iteration loop (48), whose parallel execution is wrong -- as it would be
# with an OpenACC compiler.
FT_EXACT = [0, 3, 4, 10, 13, 16, 19, 22, 25, 28, 31, 34, 37, 40, 43, 45, 49, 53, 56, 59,
            62, 65, 68, 71, 74, 77, 80, 83, 86, 88, 91]      # no two nested
FT_EXACT_SINGLE = FT_EXACT + [5]                           # 5: inside 4
FT_WRONG = [6, 7, 9, 12, 21, 24, 33, 36, 48, 52, 55, 64, 67, 76, 79]


def _genome(ev, on):
    return tuple(int(l in on) for l in ev.eligible_ids)


@pytest.mark.gpu
def test_ft_exact_loops_on_gpu_verify(gpu):
    with generic.GenEvaluator("ft_s", devices=[0]) as ev:
        g = _genome(ev, FT_EXACT)
        m = ev.measure(g)
        assert m.seconds is not None, m
        st = ev.stats[g]
        assert st["n_launch"] > 0
        assert ft.checksum_error(ev.outputs[g], "S") <= 1e-9, ev.outputs[g]


@pytest.mark.gpu
def test_ft_every_single_gene_runs(gpu):
    """Each eligible loop alone on the GPU: runs (no device fault); the exact ones verify."""
    with generic.GenEvaluator("ft_s", devices=[0]) as ev:
        for lid in ev.eligible_ids:
            g = _genome(ev, [lid])
            m = ev.measure(g)
            assert m.seconds is not None, (lid, m)
            err = ft.checksum_error(ev.outputs[g], "S")
            if lid in FT_EXACT_SINGLE:
                assert err <= 1e-9, (lid, err)


@pytest.mark.gpu
def test_ft_verify_each_rejects_wrong_patterns(gpu):
    # loops whose device result is deterministically wrong (carried scalar chains, FFT
    # stage loops); the racy line-batch loops can come out right by timing and are
    # rejected statically by the probe instead (test_ft_execution_probe)
    with generic.GenEvaluator("ft_s", devices=[0], verify_each=True) as ev:
        for lid in (6, 7, 12, 24, 36):
            m = ev.measure(_genome(ev, [lid]))
            assert m.failure and "differs" in m.failure, (lid, m)
        m = ev.measure(_genome(ev, FT_EXACT))
        assert m.seconds is not None, m


@pytest.mark.gpu
def test_generated_himeno_matches_hand_written(gpu):
    from paper_2002_12115_b200.evaluator import B200Evaluator
    # (genomes with gene 6 are excluded: the hand-written library runs the time loop as one
    # sequential device-resident loop; the generated executor
    # follows `parallel loop` literally)
    genomes = ["0000000100100", "0010010010010", "1001000100100", "1000000001100",
               "0100100100010"]
    with generic.GenEvaluator("himeno_xs", devices=[0]) as gen, \
            B200Evaluator("XS", nn=3, devices=[0]) as hand:
        for s in genomes:
            g = tuple(int(c) for c in s)
            a = gen.run_for_output(g).split()
            b = hand.run_for_output(g, literal_gosa=False).split()   # fp32(fp64 sum), as gen
            assert a[1:] == b[1:], (s, a, b)                 # p samples bit-exact
            assert abs(float(a[0]) - float(b[0])) <= 1e-5 * float(b[0]), (s, a[0], b[0])


@pytest.mark.gpu
def test_run_ga_on_ft(gpu):
    from paper_2002_12115_b200 import ga
    with generic.GenEvaluator("ft_s", devices=[0], workers_per_device=2, verify_each=True) as ev:
        res = ga.run_ga(ga.GAConfig(population=6, generations=3, rng_seed=0), ev.gene_length, ev)
        assert res.evaluations > 0 and res.best.time_s > 0


@pytest.mark.gpu
def test_ft_execution_probe(gpu):
    """The execution probe keeps every exact loop and drops the static probe's false accepts."""
    with generic.GenEvaluator("ft_s", devices=[0], genes="verified",
                              nested_policy="outermost", verify_each=True) as ev:
        kept = set(ev.eligible_ids)
        assert set(FT_EXACT_SINGLE) <= kept, set(FT_EXACT_SINGLE) - kept
        assert not (set(FT_WRONG) & kept)
        assert all(ev.probe_log[l].startswith("verified") for l in kept)
        from paper_2002_12115_b200 import ga
        res = ga.run_ga(ga.GAConfig(population=6, generations=2, rng_seed=1), ev.gene_length, ev)
        assert res.best.time_s < 1000          # verified patterns only: a runnable best


@pytest.mark.gpu
def test_ft_class_a_exact_pattern_verifies_and_beats_cpu(gpu):
    """Class A (256x256x128): the exact loops on the B200 reproduce NPB's checksums and run
    faster than the all-CPU program."""
    with generic.GenEvaluator("ft_a", devices=[0]) as ev:
        prog = ft.program("A")
        exact = [l for l in ev.eligible_ids if l in _ft_exact_ids(prog)]
        g = _genome(ev, exact)
        m = ev.measure(g)
        assert m.seconds is not None, m
        assert ft.checksum_error(ev.outputs[g], "A") <= 1e-9
        cpu = ev.measure((0,) * ev.gene_length)
        assert m.seconds < cpu.seconds, (m.seconds, cpu.seconds)


def _ft_exact_ids(prog):
    """Loops of an FT program whose device version is exact and which are not nested in
    one another: collapsed kernels nests and gang loops with vector leaves, per the
    structure of apps/ft.py (twiddle, seeds, plane fill, every copy / butterfly / evolve /
    checksum loop)."""
    from paper_2002_12115_b200 import codegen
    p = codegen.CProgram(ft.source_text(prog.cls))
    loops = prog.model.loops
    out = []
    for l in loops:
        if l.loop_id not in prog.eligible:
            continue
        anc = loops.ancestors(l.loop_id)[1:]
        if any(a in out for a in anc):
            continue
        kp = codegen.plan_kernel(p, l, prog.kinds[l.loop_id].value, loops, {k: v.value for k, v in prog.kinds.items()})
        if kp is None or (kp.carried and kp.mode != "seq") or codegen.shared_writes(p, l):
            continue
        # FFT stage loops (l) carry data between iterations through the scratch rows
        if l.index_var == "l" or l.index_var == "it":
            continue
        out.append(l.loop_id)
    return out


@pytest.mark.gpu
def test_generated_himeno_random_patterns_match_hand_written(gpu):
    """20 random runnable Himeno patterns (no gene 6, whose semantics differ by design):
    generated and hand-written executors print the same p samples bit for bit."""
    from paper_2002_12115_b200.evaluator import B200Evaluator, valid_genomes
    prog = himeno.program()
    pool = [g for g in valid_genomes(prog.model.loops, list(prog.eligible)) if not g[6]]
    rng = random.Random(11)
    with generic.GenEvaluator("himeno_xs", devices=[0]) as gen, \
            B200Evaluator("XS", nn=3, devices=[0]) as hand:
        for g in rng.sample(pool, 20):
            a = gen.run_for_output(g).split()
            b = hand.run_for_output(g, literal_gosa=False).split()   # fp32(fp64 sum), as gen
            assert a[1:] == b[1:], (g, a, b)
            # gosa: the generated executor's host stencil sums ss*ss in fp32 as the C
            # program does, the hand-written library in fp64 (B.5): at
            # XS the two differ by 0.04 %
            assert abs(float(a[0]) - float(b[0])) <= 1e-3 * float(b[0]), (g, a[0], b[0])


# ------------------------------------------------------------------ ABI (app_b200.h)

def _declared_hpg():
    import re
    from conftest import ROOT
    body = re.sub(r"/\*.*?\*/", "", (ROOT / "include" / "app_b200.h").read_text(), flags=re.S)
    return sorted(set(re.findall(r"\b(hpg_[a-z_0-9]+)\s*\(", body)))


@pytest.mark.parametrize("app", generic.APPS)
def test_generated_library_exports_every_declared_symbol(app):
    lib = generic.load(app).lib
    names = _declared_hpg()
    assert "hpg_run" in names and "hpg_create" in names
    for name in names:
        assert hasattr(lib, name), name
    assert set(names) <= set(generic.SIGNATURES)


def test_generated_struct_layouts_match_header(tmp_path):
    import ctypes as C
    import subprocess
    from conftest import ROOT
    structs = {"hpg_event": generic.Event, "hpg_schedule": generic.Schedule,
               "hpg_result": generic.Result}
    lines = ["#include <stdio.h>", "#include <stddef.h>", '#include "app_b200.h"',
             "int main(void) {"]
    for cname, py in structs.items():
        lines.append(f'  printf("{cname} size %zu\\n", sizeof({cname}));')
        for fname, _ in py._fields_:
            lines.append(f'  printf("{cname} {fname} %zu\\n", offsetof({cname}, {fname}));')
    lines += ["  return 0;", "}"]
    src = tmp_path / "probe.c"
    src.write_text("\n".join(lines) + "\n")
    subprocess.run(["gcc", "-I", str(ROOT / "include"), str(src), "-o", str(tmp_path / "p")],
                   check=True)
    got = {}
    out = subprocess.run([str(tmp_path / "p")], capture_output=True, text=True, check=True).stdout
    for line in out.splitlines():
        cname, field, value = line.split()
        got[(cname, field)] = int(value)
    for cname, py in structs.items():
        assert got[(cname, "size")] == C.sizeof(py), cname
        for fname, _ in py._fields_:
            assert got[(cname, fname)] == getattr(py, fname).offset, (cname, fname)


def _build_c_app(tmp_path):
    import subprocess
    from conftest import ROOT
    lib_dir = ROOT / "paper_2002_12115_b200" / "_native"
    exe = tmp_path / "c_app"
    subprocess.run(["gcc", "-std=c11", "-Wall", "-Werror", "-I", str(ROOT / "include"),
                    str(ROOT / "tests" / "c_app_example.c"), str(lib_dir / "libapp_ft_s.so"),
                    f"-Wl,-rpath,{lib_dir}", "-o", str(exe)], check=True)
    return exe


def test_c_host_runs_generated_ft_on_cpu(tmp_path):
    """A plain C program drives libapp_ft_s.so (host-only context): NPB checksums."""
    import subprocess
    out = subprocess.run([str(_build_c_app(tmp_path))], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout + out.stderr
    assert out.stdout == (GOLDEN / "ft_s.stdout").read_text()


@pytest.mark.gpu
def test_c_host_runs_generated_ft_on_gpu(gpu, tmp_path):
    import subprocess
    out = subprocess.run([str(_build_c_app(tmp_path)), "gpu"], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout + out.stderr
    assert ft.checksum_error(out.stdout, "S") <= 1e-9
    assert "1 launches" in out.stderr or "launches" in out.stderr


@pytest.mark.gpu
def test_ft_screened_genes(gpu):
    """genes="screened": verified loops that alone are no slower than the all-CPU program."""
    with generic.GenEvaluator("ft_s", devices=[0], genes="screened",
                              nested_policy="outermost", verify_each=True) as ev:
        cpu = ev.probe_times["cpu"]
        assert 0 < ev.gene_length < 64
        for lid in ev.eligible_ids:
            assert ev.probe_log[lid].startswith("verified")
            assert ev.probe_times[lid] <= 1.05 * cpu


@pytest.mark.gpu
def test_tune_pipeline_on_ft(gpu, tmp_path):
    """The tuning pipeline (baseline, GA, verify_results, reports) on a generated executor."""
    from paper_2002_12115_b200 import tune
    rc = tune.main(["--app", "ft_s", "--genes", "screened", "--population", "6",
                    "--generations", "2", "--out", str(tmp_path)])
    assert rc == 0
    import json
    rep = json.loads((tmp_path / "report.json").read_text())
    assert rep["verification"]["status"] == "ran" and rep["verification"]["passed"]


@pytest.mark.gpu
def test_ft_random_verified_patterns_reproduce_npb(gpu):
    """Random combinations of verified loops (nested genes under their outermost anchor):
    every run reproduces NPB's checksums -- the data manager's hoisted transfers, dirty
    boxes and staging are exact in combination, not only per loop."""
    with generic.GenEvaluator("ft_s", devices=[0], genes="verified",
                              nested_policy="outermost") as ev:
        rng = random.Random(2002)
        for _ in range(16):
            g = tuple(rng.randint(0, 1) for _ in range(ev.gene_length))
            m = ev.measure(g)
            assert m.seconds is not None, m
            assert ft.checksum_error(ev.outputs[g], "S") <= 1e-9, (g, ev.outputs[g])


@pytest.mark.gpu
def test_ft_class_w_exact_pattern(gpu):
    with generic.GenEvaluator("ft_w", devices=[0]) as ev:
        exact = _ft_exact_ids(ft.program("W"))
        g = _genome(ev, [l for l in ev.eligible_ids if l in exact])
        m = ev.measure(g)
        assert m.seconds is not None, m
        assert ft.checksum_error(ev.outputs[g], "W") <= 1e-9


@pytest.mark.gpu
def test_ft_per_loop_plan_is_wrong_for_evolve(gpu):
    """The reference's raw per-loop directions give the evolve loop (49) u0 `copyin`
    only, so its device update never returns: the batched plan verifies,
    the per-loop one does not -- as an OpenACC build of those directives would."""
    for mode, ok in (("batched", True), ("per-loop", False)):
        with generic.GenEvaluator("ft_s", devices=[0], transfer_mode=mode) as ev:
            g = _genome(ev, [49])
            m = ev.measure(g)
            assert m.seconds is not None, m
            assert (ft.checksum_error(ev.outputs[g], "S") <= 1e-9) == ok, mode
