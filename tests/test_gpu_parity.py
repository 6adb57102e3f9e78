"""GPU parity: the native B200 path against the CPU oracle (run on a B200 box).

Bar: p is bit-exact (every product/sum is rounded
separately on both sides, no FMA); gosa is an fp64 sum of the same fp32 terms
in a different order, so |gosa - oracle_fp64| <= 1e-12 * oracle_fp64 -- far
inside north_star's 1e-5.
"""
import numpy as np
import pytest

from oracle import oracle
from paper_2002_12115_b200 import native as N
from paper_2002_12115_b200.apps import himeno
from paper_2002_12115_b200.evaluator import B200Evaluator, MeasuredTime, valid_genomes
from paper_2002_12115_b200.errors import TunerError
from paper_2002_12115_b200.kinds import DirectiveKind

pytestmark = pytest.mark.gpu
GOSA_RTOL = 1e-12

_ORACLE = {}


def oracle_result(name, nn):
    key = (name, nn)
    if key not in _ORACLE:
        sz = himeno.size(name)
        _ORACLE[key] = oracle.run_program(sz.I, sz.J, sz.K, nn)
    return _ORACLE[key]


def check_run(ev, genome, ref):
    res = ev.run(genome)
    assert res.status == 0, res.diag
    p = ev.read_field("p", side=0)
    assert np.array_equal(p, ref["fields"]["p"]), f"p differs for {genome}"
    assert abs(res.gosa - ref["gosa64"]) <= GOSA_RTOL * ref["gosa64"], (genome, res.gosa)
    assert res.n_stale_reads == 0, (genome, res.stats())
    return res


@pytest.fixture(scope="module")
def ev_xs(gpu):
    ev = B200Evaluator("XS", nn=3, poison_device=True)
    yield ev
    ev.close()


def test_all_cpu_and_best_patterns(ev_xs):
    ref = oracle_result("XS", 3)
    for g in ["0000000000000", "0000000100100", "0000001000000", "1001001000000",
              "0010010010010", "0100100100100"]:
        check_run(ev_xs, tuple(int(c) for c in g), ref)


def test_every_valid_genome_xs(ev_xs):
    """All 272 non-nested Himeno genomes reproduce the all-CPU output exactly."""
    ref = oracle_result("XS", 3)
    genomes = valid_genomes(ev_xs.loops, ev_xs.eligible_ids)
    assert len(genomes) == 272
    for g in genomes:
        check_run(ev_xs, g, ref)


def test_stdout_matches_reference_tokens(ev_xs):
    out = ev_xs.run_for_output((0, 0, 0, 0, 0, 0, 1, 0, 0, 0, 0, 0, 0)).split()
    want = open("tests/golden/himeno_xs_n3.stdout").read().split()
    assert out[1:] == want[1:]                      # p samples: exact
    assert abs(float(out[0]) - float(want[0])) / float(want[0]) < 1e-3  # fp32-seq drift


def test_nested_pattern_rejected_before_launch(ev_xs):
    m = ev_xs.measure((0, 0, 0, 0, 0, 0, 1, 1, 0, 0, 0, 0, 0))
    assert m.failure and "nested" in m.failure


def test_per_loop_transfer_mode_moves_more(gpu):
    ref = oracle_result("XS", 3)
    g = (0, 0, 0, 0, 0, 0, 0, 1, 0, 0, 1, 0, 0)
    with B200Evaluator("XS", nn=3, transfer_mode="per-loop") as raw, \
            B200Evaluator("XS", nn=3) as batched:
        r1 = check_run(raw, g, ref)
        r2 = check_run(batched, g, ref)
        assert r1.h2d_bytes + r1.d2h_bytes > 2 * (r2.h2d_bytes + r2.d2h_bytes), (r1.stats(), r2.stats())
        assert r1.n_implicit > 0


def test_coherence_guard_skips_stale_update(gpu):
    # 1001001000000: update device(a, b, c, ...) at jacobi entry after device-side init
    ref = oracle_result("XS", 3)
    with B200Evaluator("XS", nn=3) as ev:
        res = check_run(ev, (1, 0, 0, 1, 0, 0, 1, 0, 0, 0, 0, 0, 0), ref)
        assert res.n_skipped_stale > 0


@pytest.mark.parametrize("kind", [DirectiveKind.PARALLEL_LOOP, DirectiveKind.PARALLEL_LOOP_VECTOR])
def test_alternative_kinds(gpu, kind):
    ref = oracle_result("XXS", 3)
    prog = himeno.program()
    kinds = {lid: kind for lid in prog.kinds}
    with B200Evaluator("XXS", nn=3, kinds=kinds) as ev:
        for g in ["0000000100100", "0100100100100", "0010010010010", "1001001000000",
                  "0000001000000"]:
            check_run(ev, tuple(int(c) for c in g), ref)


def test_unfused_time_loop(gpu):
    ref = oracle_result("XS", 3)
    with B200Evaluator("XS", nn=3, fused_time_loop=False) as ev:
        check_run(ev, (0, 0, 0, 0, 0, 0, 1, 0, 0, 0, 0, 0, 0), ref)


def test_timeout_maps_to_measured_timeout(gpu):
    with B200Evaluator("S", nn=50, timeout_s=0.05) as ev:
        m = ev.measure((0,) * 13)
        assert m == MeasuredTime.timeout()


@pytest.mark.parametrize("variant", [0, 1])
@pytest.mark.parametrize("name,nn", [("XS", 3), ("M", 2)])
def test_device_jacobi_variants(gpu, variant, name, nn):
    ref = oracle_result(name, nn)
    sz = himeno.size(name)
    with N.Context(0, sz.I, sz.J, sz.K) as ctx:
        ctx.init_device()
        ctx.jacobi_device(nn, variant)
        g = ctx.read_gosa(1)
        p = ctx.read_field("p", 1)
        w = ctx.read_field("wrk2", 1)
    assert np.array_equal(p, ref["fields"]["p"])
    assert np.array_equal(w, ref["fields"]["wrk2"])
    assert abs(g - ref["gosa64"]) <= GOSA_RTOL * ref["gosa64"]


def test_jacobi_host_e2e(gpu):
    name, nn = "S", 2
    sz = himeno.size(name)
    f = oracle.empty_fields(sz.I, sz.J, sz.K)
    oracle.initmt(f)
    inputs = {k: v.copy() for k, v in f.items()}
    g64, _ = oracle.jacobi(f, nn)
    p_out = np.empty_like(f["p"])
    with N.Context(0, sz.I, sz.J, sz.K) as ctx:
        g = ctx.jacobi_host(inputs, nn, 1, p_out)
    assert np.array_equal(p_out, f["p"])
    assert abs(g - g64) <= GOSA_RTOL * g64


def test_jacobi_host_async_pipeline(gpu):
    """Two contexts alternating hp_jacobi_host_async jobs (the bench e2e pipeline) give
    the serial call's results; a second async call before hp_sync is refused."""
    name, nn = "S", 3
    sz = himeno.size(name)
    f = oracle.empty_fields(sz.I, sz.J, sz.K)
    oracle.initmt(f)
    inputs = {k: v.copy() for k, v in f.items()}
    g64, _ = oracle.jacobi(f, nn)
    outs = [np.empty_like(f["p"]), np.empty_like(f["p"])]
    with N.Context(0, sz.I, sz.J, sz.K) as a, N.Context(0, sz.I, sz.J, sz.K) as b:
        ctxs, got = (a, b), []
        for step in range(5):
            x = step % 2
            if step >= 2:
                got.append(ctxs[x].sync())
            ctxs[x].jacobi_host_async(inputs, nn, 1, outs[x])
        with pytest.raises(TunerError):
            ctxs[0].jacobi_host_async(inputs, nn, 1, outs[0])
        got += [a.sync(), b.sync()]
        assert a.sync() is None
    assert len(got) == 5
    for g in got:
        assert abs(g - g64) <= GOSA_RTOL * g64
    for out in outs:
        assert np.array_equal(out, f["p"])


def test_gosa_bit_reproducible_under_concurrency(gpu):
    """gosa of the unit-queue kernels is folded per work unit in unit order, so it is
    bit-identical whichever CTA ran which unit: alone, and with a second context's
    kernels competing for the SMs."""
    sz = himeno.size("M")
    with N.Context(0, sz.I, sz.J, sz.K) as a, N.Context(0, sz.I, sz.J, sz.K) as b:
        ref = None
        for tb in (1, 0):
            lib = a.lib
            old = lib.hp_set_temporal_blocking(tb)
            try:
                got = []
                a.init_device()
                a.jacobi_device(6, 1)
                got.append(a.read_gosa(1))
                for _ in range(3):
                    a.init_device()
                    b.init_device()
                    b.jacobi_device(9, 1)      # enqueued on b's stream: runs concurrently
                    a.jacobi_device(6, 1)
                    got.append(a.read_gosa(1))
                    b.sync()
            finally:
                lib.hp_set_temporal_blocking(old)
            assert len(set(got)) == 1, got
            if ref is None:
                ref = got[0]
            else:   # one- and two-step passes fold different units: equal to 1e-12
                assert abs(got[0] - ref) <= GOSA_RTOL * ref


def test_m_grid_selected_patterns(gpu):
    ref = oracle_result("M", 2)
    with B200Evaluator("M", nn=2) as ev:
        for g in ["0000000100100", "1001001000000", "0000001000000", "1001000100100"]:
            check_run(ev, tuple(int(c) for c in g), ref)


@pytest.mark.parametrize("name,nn", [("XS", 2), ("M", 2), ("custom", 3)])
def test_every_stencil_config_bit_exact(gpu, name, nn):
    """Register and TMA stencil variants all reproduce the oracle exactly."""
    sz = himeno.custom_size(37, 21, 70) if name == "custom" else himeno.size(name)
    ref = oracle.run_program(sz.I, sz.J, sz.K, nn)
    lib = N.load()
    ncfg = lib.hp_set_stencil_config(0)
    try:
        with N.Context(0, sz.I, sz.J, sz.K) as ctx:
            for cfg in range(ncfg):
                assert lib.hp_set_stencil_config(cfg) == ncfg
                for variant in (0, 1):
                    ctx.init_device()
                    ctx.jacobi_device(nn, variant)
                    p = ctx.read_field("p", 1)
                    g = ctx.read_gosa(1)
                    assert np.array_equal(p, ref["fields"]["p"]), (cfg, variant)
                    assert abs(g - ref["gosa64"]) <= GOSA_RTOL * ref["gosa64"], (cfg, variant)
    finally:
        lib.hp_set_stencil_config(7)


@pytest.mark.parametrize("shape", [0, 1, 2, 3])
@pytest.mark.parametrize("chunk", [0, 16, 40])
def test_two_step_shapes_bit_exact(gpu, monkeypatch, shape, chunk):
    """Every compiled two-step tile shape, at the scheduler's unit length and at pinned
    ones (HIMENO_TB2_SHAPE / HIMENO_TB2_CHUNK are read per launch), on a ragged grid whose
    k and j extents are not multiples of any tile."""
    sz = himeno.custom_size(75, 45, 141)
    nn = 4
    ref = oracle.run_program(sz.I, sz.J, sz.K, nn)
    monkeypatch.setenv("HIMENO_TB2_SHAPE", str(shape))
    if chunk:
        monkeypatch.setenv("HIMENO_TB2_CHUNK", str(chunk))
    lib = N.load()
    old = lib.hp_set_temporal_blocking(1)
    try:
        with N.Context(0, sz.I, sz.J, sz.K) as ctx:
            ctx.init_device()
            ctx.jacobi_device(nn, 1)
            p, g = ctx.read_field("p", 1), ctx.read_gosa(1)
            kt = ctx.time_jacobi(nn, 1)
    finally:
        lib.hp_set_temporal_blocking(old)
    assert kt.stencil_iters >= 2.0     # two-step passes (one flow launch of both, or two)
    assert np.array_equal(p, ref["fields"]["p"])
    assert abs(g - ref["gosa64"]) <= GOSA_RTOL * ref["gosa64"]


@pytest.mark.parametrize("stash", [0, 1])
@pytest.mark.parametrize("full", [0, 2, 5, 9])
def test_two_step_whole_columns_bit_exact(gpu, monkeypatch, full, stash):
    """Whole tile columns ahead of the chunked tail (HIMENO_TB2_FULL pins how many; the
    grid has 3 x 3 tiles of shape (16,8,4), so 9 = every tile a whole column) give the
    same field, bit for bit, as the oracle -- with the step-2 coefficients stashed in
    tensor memory (the default) and read from the shared-memory stage."""
    sz = himeno.custom_size(75, 45, 141)
    nn = 4
    ref = oracle.run_program(sz.I, sz.J, sz.K, nn)
    monkeypatch.setenv("HIMENO_TB2_SHAPE", "1")
    monkeypatch.setenv("HIMENO_TB2_CHUNK", "16")
    monkeypatch.setenv("HIMENO_TB2_FULL", str(full))
    monkeypatch.setenv("HIMENO_TB2_STASH", str(stash))
    lib = N.load()
    old = lib.hp_set_temporal_blocking(1)
    try:
        with N.Context(0, sz.I, sz.J, sz.K) as ctx:
            ctx.init_device()
            ctx.jacobi_device(nn, 1)
            p, g = ctx.read_field("p", 1), ctx.read_gosa(1)
            kt = ctx.time_jacobi(nn, 1)
    finally:
        lib.hp_set_temporal_blocking(old)
    assert kt.stencil_iters >= 2.0     # two-step passes (one flow launch of both, or two)
    assert np.array_equal(p, ref["fields"]["p"])
    assert abs(g - ref["gosa64"]) <= GOSA_RTOL * ref["gosa64"]


@pytest.mark.parametrize("tb", [0, 1])
@pytest.mark.parametrize("name,nn", [("XS", 1), ("XS", 4), ("XS", 5), ("M", 2), ("M", 3),
                                      ("custom", 4), ("ragged", 3)])
def test_temporal_blocking_bit_exact(gpu, tb, name, nn):
    """Two-step passes (temporal blocking) reproduce nn single iterations exactly."""
    if name == "custom":
        sz = himeno.custom_size(37, 21, 70)
    elif name == "ragged":
        sz = himeno.custom_size(20, 29, 300)
    else:
        sz = himeno.size(name)
    ref = oracle.run_program(sz.I, sz.J, sz.K, nn)
    lib = N.load()
    old = lib.hp_set_temporal_blocking(tb)
    try:
        with N.Context(0, sz.I, sz.J, sz.K) as ctx:
            ctx.init_device()
            ctx.jacobi_device(nn, 1)
            p, w, g = ctx.read_field("p", 1), ctx.read_field("wrk2", 1), ctx.read_gosa(1)
            kt = ctx.time_jacobi(nn, 1)
    finally:
        lib.hp_set_temporal_blocking(old)
    assert np.array_equal(p, ref["fields"]["p"])
    assert np.array_equal(w, ref["fields"]["wrk2"])
    assert abs(g - ref["gosa64"]) <= GOSA_RTOL * ref["gosa64"]
    if tb and nn >= 2:
        assert kt.stencil_iters > 1.0


def test_concurrent_workers_share_a_device(gpu):
    """Population sharding with several worker slots (own contexts) on one GPU."""
    from concurrent.futures import ThreadPoolExecutor
    ref = oracle_result("XS", 3)
    with B200Evaluator("XS", nn=3, workers_per_device=3) as ev:
        assert ev.max_concurrency == 3
        genomes = valid_genomes(ev.loops, ev.eligible_ids)[::23]
        with ThreadPoolExecutor(max_workers=3) as pool:
            results = list(pool.map(ev.measure, genomes))
        assert all(m.seconds for m in results)
        for g in genomes:
            st = ev.stats[g]
            assert abs(st["gosa"] - ref["gosa64"]) <= GOSA_RTOL * ref["gosa64"], g
            assert st["n_stale_reads"] == 0
        assert len(ev._contexts) == 3


@pytest.mark.parametrize("tb", [0, 1])
def test_headline_L_grid_bit_exact(gpu, tb):
    """The bench workload's grid (L), both time-loop kernels, against the oracle."""
    sz = himeno.size("L")
    nn = 3
    f = oracle.empty_fields(sz.I, sz.J, sz.K)
    oracle.initmt(f)
    g64, _ = oracle.jacobi(f, nn, threads=oracle.max_threads())
    lib = N.load()
    old = lib.hp_set_temporal_blocking(tb)
    try:
        with N.Context(0, sz.I, sz.J, sz.K) as ctx:
            ctx.init_device()
            ctx.jacobi_device(nn, 1)
            p, g = ctx.read_field("p", 1), ctx.read_gosa(1)
    finally:
        lib.hp_set_temporal_blocking(old)
    assert np.array_equal(p, f["p"])
    assert abs(g - g64) <= 1e-11 * g64     # threaded oracle sums planes in another order


@pytest.mark.parametrize("dims", [(4, 4, 4), (5, 4, 9), (4, 7, 5), (6, 6, 6), (9, 5, 133)])
def test_tiny_and_ragged_grids_all_genomes(gpu, dims):
    """Minimal / ragged grids (one interior point, partial tiles) for every runnable genome."""
    sz = himeno.custom_size(*dims)
    for nn in (1, 2, 3):
        ref = oracle.run_program(sz.I, sz.J, sz.K, nn)
        with B200Evaluator(sz, nn=nn, poison_device=True) as ev:
            for g in valid_genomes(ev.loops, ev.eligible_ids)[::7]:
                res = ev.run(g)
                p = ev.read_field("p", side=0)
                assert np.array_equal(p, ref["fields"]["p"]), (dims, nn, g)
                assert abs(res.gosa - ref["gosa64"]) <= GOSA_RTOL * max(ref["gosa64"], 1e-300), \
                    (dims, nn, g, res.gosa, ref["gosa64"])


@pytest.mark.parametrize("tb", [0, 1])
def test_device_jacobi_zero_iterations(gpu, tb):
    sz = himeno.size("XS")
    ref = oracle.run_program(sz.I, sz.J, sz.K, 0)
    lib = N.load()
    old = lib.hp_set_temporal_blocking(tb)
    try:
        with N.Context(0, sz.I, sz.J, sz.K) as ctx:
            ctx.init_device()
            ctx.jacobi_device(0, 1)
            assert np.array_equal(ctx.read_field("p", 1), ref["fields"]["p"])
    finally:
        lib.hp_set_temporal_blocking(old)


# --- main's printed float gosa (hp_result.gosa_f32) ---------------------------------------

GOLDEN_STDOUT = [("XXS", 1), ("XXS", 3), ("XS", 1), ("XS", 3), ("S", 2), ("M", 2)]


@pytest.mark.parametrize("name,nn", GOLDEN_STDOUT)
def test_host_stencil_stdout_equals_reference_program(gpu, name, nn):
    """With the stencil nest on the host, the B200 program prints exactly what the
    reference's own ExternalEvaluator.run_for_output printed for the same program
    (tests/golden/*.stdout, oracle/pin_reference.py): the literal fp32 sequential
    gosa, byte for byte -- also when other nests run on the device."""
    from conftest import GOLDEN
    want = (GOLDEN / f"himeno_{name.lower()}_n{nn}.stdout").read_text()
    with B200Evaluator(name, nn=nn, poison_device=True) as ev:
        for g in ("0000000000000", "0000000000100", "1001000000000"):
            genome = tuple(int(c) for c in g)
            assert ev.run_for_output(genome, literal_gosa=False) == want, (name, nn, g)
            assert ev.stats[genome]["gosa_f32_literal"], g
        # stencil on the device (kernels / gang rows / the device time loop, fused and
        # two-step): verification mode sums the pattern's own device terms in order
        for g in ("0000000100100", "0000000001001", "0000001000000", "1001001000000",
                  "0100100100100"):
            genome = tuple(int(c) for c in g)
            assert ev.run_for_output(genome) == want, (name, nn, g)
            assert ev.stats[genome]["gosa_f32_literal"], g


def test_device_stencil_gosa_f32_is_rounded_fp64(gpu):
    with B200Evaluator("XS", nn=3) as ev:
        for g in ("0000000100100", "0000001000000"):
            genome = tuple(int(c) for c in g)
            res = ev.run(genome)
            assert not res.gosa_f32_literal
            assert res.gosa_f32 == np.float32(res.gosa)


def test_smem_optin_raised_on_every_device_used(gpu):
    """The large-shared-memory kernels' opt-in is set per device context (a
    process-wide flag would leave devices 1..7 without it)."""
    with B200Evaluator("M", nn=4, devices="all") as ev:
        ev.prepare()
        for slot in range(ev.max_concurrency):
            ev._context(slot)   # noqa: SLF001 - every device gets a context
        for dev in sorted(set(ev.devices)):
            # run the time-loop pattern on that device (two-step + single-step kernels)
            ctx = ev._contexts[ev.devices.index(dev)]
            ctx.init_device()
            ctx.jacobi_device(3, 1)
            ctx.sync()
            # two-step kernel (cross-warp stash, coefficients-first order: M's planes fit L2)
            assert N.smem_optin(12, dev) > 48 * 1024, dev
            assert N.smem_optin(1, dev) > 48 * 1024, dev   # single-step, 3 stages


# --- BASELINE configs at full size ----------------------------------------------------------

def test_headline_L_bench_step_matches_golden(gpu):
    """The bench's step (L, jacobi(100), device time loop with two-step passes) against
    the oracle's committed result (scripts/gen_golden_l100.py): p bit-exact (SHA-256 of
    the field), gosa within 1e-11."""
    import hashlib
    import json
    from conftest import GOLDEN
    want = json.loads((GOLDEN / "himeno_l_n100.json").read_text())
    sz = himeno.size("L")
    with N.Context(0, sz.I, sz.J, sz.K) as ctx:
        ctx.init_device()
        ctx.jacobi_device(want["nn"], 1)
        p, g = ctx.read_field("p", 1), ctx.read_gosa(1)
    assert hashlib.sha256(p.tobytes()).hexdigest() == want["p_sha256"]
    assert abs(g - want["gosa64"]) <= 1e-11 * want["gosa64"]
    for i, j, k, v in want["p_samples"]:
        assert p[i, j, k] == np.float32(v)


@pytest.fixture(scope="module")
def xl_oracle():
    """XL (config 5's grid) after 2 and after 4 iterations, threaded oracle."""
    sz = himeno.size("XL")
    f = oracle.empty_fields(sz.I, sz.J, sz.K)
    oracle.initmt(f)
    out = {}
    g2, _ = oracle.jacobi(f, 2, threads=oracle.max_threads())
    out[2] = (f["p"].copy(), g2)
    g4, _ = oracle.jacobi(f, 2, threads=oracle.max_threads())   # iterations 3-4
    out[4] = (f["p"], g4)
    for name in list(f):
        if name != "p":
            del f[name]
    return out


@pytest.mark.parametrize("tb", [0, 1])
def test_xl_grid_bit_exact(gpu, xl_oracle, tb):
    """XL 513x513x1025 (BASELINE config 5), one- and two-step kernels, nn = 2 and 4."""
    sz = himeno.size("XL")
    lib = N.load()
    old = lib.hp_set_temporal_blocking(tb)
    try:
        with N.Context(0, sz.I, sz.J, sz.K) as ctx:
            for nn in (2, 4):
                ctx.init_device()
                ctx.jacobi_device(nn, 1)
                p, g = ctx.read_field("p", 1), ctx.read_gosa(1)
                want_p, want_g = xl_oracle[nn]
                assert np.array_equal(p, want_p), (tb, nn)
                assert abs(g - want_g) <= 1e-11 * want_g, (tb, nn, g, want_g)
                del p
    finally:
        lib.hp_set_temporal_blocking(old)


@pytest.fixture(scope="module")
def l_oracle_n4():
    sz = himeno.size("L")
    f = oracle.empty_fields(sz.I, sz.J, sz.K)
    oracle.initmt(f)
    g3, _ = oracle.jacobi(f, 3, threads=oracle.max_threads())
    p3 = f["p"].copy()
    g4, _ = oracle.jacobi(f, 1, threads=oracle.max_threads())
    return {3: (p3, g3), 4: (f["p"].copy(), g4)}


@pytest.mark.parametrize("overlap", [0, 1, 2])
@pytest.mark.parametrize("tb", [0, 1])
@pytest.mark.parametrize("ranks", [2, 4, 8])
def test_l_grid_slabs_bit_exact(gpu, monkeypatch, l_oracle_n4, ranks, tb, overlap):
    """BASELINE config 3's decomposition (L split into 2/4/8 slabs, halo exchange --
    after each pass, or overlapped with the interior: boundary planes first, exchange on
    a comm stream -- and gosa sum after the passes) with virtual ranks on one GPU,
    against the full grid."""
    from paper_2002_12115_b200 import dd
    # 0: exchange after each whole pass; 1: overlapped, one launch whose boundary units
    # signal the exchange stream; 2: overlapped as two launches (boundary, interior)
    monkeypatch.setenv("HIMENO_DD_OVERLAP", str(min(overlap, 1)))
    monkeypatch.setenv("HIMENO_DD_SIGNAL", "0" if overlap == 2 else "1")
    lib = N.load()
    old = lib.hp_set_temporal_blocking(tb)
    try:
        for nn in (3, 4):
            with dd.GroupJacobi("L", [0] * ranks) as g:
                gosa = g.jacobi(nn)
                p = g.gather("p")
            want_p, want_g = l_oracle_n4[nn]
            assert np.array_equal(p, want_p), (ranks, tb, nn)
            assert abs(gosa - want_g) <= 1e-11 * want_g, (ranks, tb, nn)
    finally:
        lib.hp_set_temporal_blocking(old)


# --- the tile-exchange two-step kernel (k_stencil_tx) ----------------------------------

@pytest.mark.parametrize("dims,nn,minchunk", [
    ((75, 45, 141), 4, 0),     # 2 x 6 tiles, ragged j and k
    ((75, 45, 141), 5, 8),     # several plane chunks, odd nn (one single-step pass)
    ((37, 21, 70), 4, 4),      # one k-tile, 3 j-tiles, 4-plane chunks
    ((20, 17, 300), 3, 4),     # 3 k-tiles, j extent a multiple of the tile rows
    ((6, 6, 6), 2, 0),         # 3 interior planes, one tile
    ((129, 129, 257), 4, 0),   # M: 2 x 18 tiles x 4 chunks
])
def test_exchange_kernel_bit_exact(gpu, monkeypatch, dims, nn, minchunk):
    """k_stencil_tx (tiles exchange their p1 boundary through L2 instead of recomputing
    a halo) forced on small and ragged grids, several plane chunks: p bit-exact with the
    oracle, gosa within 1e-12, and the launch really was the exchange kernel."""
    sz = himeno.custom_size(*dims)
    ref = oracle.run_program(sz.I, sz.J, sz.K, nn)
    monkeypatch.setenv("HIMENO_TX", "2")
    if minchunk:
        monkeypatch.setenv("HIMENO_TX_MINCHUNK", str(minchunk))
    lib = N.load()
    old = lib.hp_set_temporal_blocking(1)
    try:
        with N.Context(0, sz.I, sz.J, sz.K) as ctx:
            ctx.init_device()
            ctx.jacobi_device(nn, 1)
            p, g = ctx.read_field("p", 1), ctx.read_gosa(1)
            assert N.last_two_step_kernel() == "k_stencil_tx"
            assert ctx.tx_status() == 0
            kt = ctx.time_jacobi(nn, 1)
    finally:
        lib.hp_set_temporal_blocking(old)
    assert kt.stencil_iters == nn / ((nn + 1) // 2)    # two-step passes + odd remainder
    assert np.array_equal(p, ref["fields"]["p"])
    assert abs(g - ref["gosa64"]) <= GOSA_RTOL * max(ref["gosa64"], 1e-300)


def test_exchange_kernel_matches_tb2_on_L(gpu, monkeypatch):
    """On the headline grid the exchange kernel's policy (HIMENO_TX=1) selects it -- 148
    tiles of 128 x 7 points, one per SM -- and it matches k_stencil_tb2 (the default,
    HIMENO_TX unset) bit for bit, with no neighbour-wait timeout."""
    sz = himeno.size("L")
    with N.Context(0, sz.I, sz.J, sz.K) as ctx:
        monkeypatch.setenv("HIMENO_TX", "1")
        ctx.init_device()
        ctx.jacobi_device(4, 1)
        assert N.last_two_step_kernel() == "k_stencil_tx"
        assert ctx.tx_status() == 0
        p_tx, g_tx = ctx.read_field("p", 1), ctx.read_gosa(1)
        monkeypatch.delenv("HIMENO_TX")
        ctx.init_device()
        ctx.jacobi_device(4, 1)
        assert N.last_two_step_kernel().startswith("k_stencil_tb2")
        p_tb, g_tb = ctx.read_field("p", 1), ctx.read_gosa(1)
    assert np.array_equal(p_tx, p_tb)
    assert abs(g_tx - g_tb) <= 1e-12 * g_tb


# --- multi-pass flow launches of the two-step kernel ----------------------------------

@pytest.mark.parametrize("dims,nn,chunk", [
    ((129, 129, 257), 100, 0),   # M, the bench's jacobi(100): 50 passes in one launch
    ((129, 129, 257), 7, 16),    # 3 passes + a single step
    ((75, 45, 141), 10, 8),      # ragged, 5 passes, 8-plane chunks (dependencies on 3 chunks)
    ((37, 21, 70), 6, 4),        # 3 passes, 4-plane chunks
    ((6, 6, 6), 4, 0),           # 3 interior planes
])
def test_flow_launch_bit_exact(gpu, monkeypatch, dims, nn, chunk):
    """Several two-step passes in one launch (units of pass t+1 wait only for their
    neighbourhood in pass t) give the oracle's field bit for bit."""
    sz = himeno.custom_size(*dims)
    if nn > 10:
        f = oracle.empty_fields(sz.I, sz.J, sz.K)
        oracle.initmt(f)
        g64, _ = oracle.jacobi(f, nn, threads=oracle.max_threads())
        ref = {"fields": f, "gosa64": g64}
        tol = 1e-11
    else:
        ref = oracle.run_program(sz.I, sz.J, sz.K, nn)
        tol = GOSA_RTOL
    monkeypatch.setenv("HIMENO_TB2_FLOW", "1")
    if chunk:
        monkeypatch.setenv("HIMENO_FLOW_CHUNK", str(chunk))
    lib = N.load()
    old = lib.hp_set_temporal_blocking(1)
    try:
        with N.Context(0, sz.I, sz.J, sz.K) as ctx:
            ctx.init_device()
            ctx.jacobi_device(nn, 1)
            assert N.last_two_step_kernel() in ("k_stencil_tb2 (flow)", "k_stencil_tb2")
            p, g = ctx.read_field("p", 1), ctx.read_gosa(1)
    finally:
        lib.hp_set_temporal_blocking(old)
    assert np.array_equal(p, ref["fields"]["p"])
    assert abs(g - ref["gosa64"]) <= tol * max(ref["gosa64"], 1e-300)


def test_flow_launch_is_the_default_on_M(gpu):
    """The device time loop on M (one pass's tiles fit in one wave) runs as a flow launch."""
    sz = himeno.size("M")
    with N.Context(0, sz.I, sz.J, sz.K) as ctx:
        ctx.init_device()
        ctx.jacobi_device(8, 1)
        assert N.last_two_step_kernel() == "k_stencil_tb2 (flow)"


# --- reference-faithful host build of the gene-0 loops ---------------------------------

@pytest.mark.parametrize("name", ["XS", "M"])
def test_host_reference_build_same_values(gpu, name):
    """host_build="reference" (the program's literal loops, g++ -O2 like the reference's
    compile template) computes exactly what the tuned host build does, for the all-CPU
    program and for mixed patterns; only its speed differs."""
    sz = himeno.size(name)
    ref = oracle.run_program(sz.I, sz.J, sz.K, 3)
    times = {}
    for build in ("tuned", "reference"):
        with B200Evaluator(name, nn=3, host_build=build) as ev:
            for g in ("0" * 13, "0000000100100", "1001000000000", "0000001000000"):
                genome = tuple(int(c) for c in g)
                res = ev.run(genome)
                p = ev.read_field("p", side=0)
                assert np.array_equal(p, ref["fields"]["p"]), (build, g)
                assert abs(res.gosa - ref["gosa64"]) <= GOSA_RTOL * ref["gosa64"], (build, g)
                if g == "0" * 13:
                    # the all-CPU program's printed float gosa: the literal fp32 sum
                    assert np.float32(res.gosa_f32) == np.float32(ref["gosa32"]), build
            times[build] = min(ev.measure((0,) * 13).seconds for _ in range(3))
    print(f"{name} all-CPU program: tuned {times['tuned'] * 1e3:.2f} ms, "
          f"reference build {times['reference'] * 1e3:.2f} ms")


# --- the new launch modes under concurrent contexts on one GPU --------------------------

@pytest.mark.parametrize("mode", ["flow", "tx"])
def test_concurrent_contexts_new_launch_modes(gpu, monkeypatch, mode):
    """Worker slots share a GPU (the GA's population sharding with several contexts per
    device): four contexts run the device time loop at once -- as multi-pass flow launches
    (CTAs wait only on units claimed earlier in their own launch), or with the tile-exchange
    kernel (its launches are chained per device across streams, so two never hold SMs the
    other needs).  Every context's field equals the oracle's; no neighbour-wait timeout."""
    from concurrent.futures import ThreadPoolExecutor
    nn = 8
    if mode == "flow":
        monkeypatch.setenv("HIMENO_TB2_FLOW", "1")
        sz = himeno.size("XS")
    else:
        monkeypatch.setenv("HIMENO_TX", "2")
        monkeypatch.setenv("HIMENO_TX_MINCHUNK", "4")
        sz = himeno.custom_size(37, 21, 70)
    ref = oracle.run_program(sz.I, sz.J, sz.K, nn)
    lib = N.load()
    old = lib.hp_set_temporal_blocking(1)
    ctxs = [N.Context(0, sz.I, sz.J, sz.K) for _ in range(4)]
    try:
        def one(c):
            out = []
            for _ in range(3):
                c.init_device()
                c.jacobi_device(nn, 1)
                out.append((c.read_field("p", 1), c.read_gosa(1), c.tx_status()))
            return out
        with ThreadPoolExecutor(max_workers=4) as pool:
            results = list(pool.map(one, ctxs))
    finally:
        for c in ctxs:
            c.close()
        lib.hp_set_temporal_blocking(old)
    for runs in results:
        for p, g, st in runs:
            assert st == 0
            assert np.array_equal(p, ref["fields"]["p"])
            assert abs(g - ref["gosa64"]) <= GOSA_RTOL * ref["gosa64"]


@pytest.mark.parametrize("overlap", [0, 1])
def test_xl_grid_8_slabs_bit_exact(gpu, monkeypatch, xl_oracle, overlap):
    """BASELINE config 5's grid (XL 513x513x1025) decomposed into 8 slabs -- virtual ranks
    on one GPU, halo exchange after each pass or overlapped with the interior -- against
    the full-grid oracle at nn = 2 and 4."""
    from paper_2002_12115_b200 import dd
    monkeypatch.setenv("HIMENO_DD_OVERLAP", str(overlap))
    for nn in (2, 4):
        with dd.GroupJacobi("XL", [0] * 8) as g:
            gosa = g.jacobi(nn)
            p = g.gather("p")
        want_p, want_g = xl_oracle[nn]
        assert np.array_equal(p, want_p), (overlap, nn)
        assert abs(gosa - want_g) <= 1e-11 * want_g, (overlap, nn)
        del p


@pytest.mark.gpu
@pytest.mark.parametrize("trim", ["0", "7"])
@pytest.mark.parametrize("kernel", ["tb2", "single", "tx"])
@pytest.mark.parametrize("dims", [(33, 33, 65), (37, 21, 70), (45, 47, 121), (20, 20, 58)])
def test_trimmed_tma_extents_bit_exact(gpu, monkeypatch, dims, kernel, trim):
    """Tensor maps ending at column K-1 / row J-1 (the default) or at K / J give the
    oracle's field bit for bit in every stencil kernel (ragged and tile-multiple grids)."""
    sz = himeno.custom_size(*dims)
    nn = 4
    ref = oracle.run_program(sz.I, sz.J, sz.K, nn)
    monkeypatch.setenv("HIMENO_TMA_TRIM", trim)
    if kernel == "tx":
        monkeypatch.setenv("HIMENO_TX", "2")
    lib = N.load()
    old = lib.hp_set_temporal_blocking(0 if kernel == "single" else 1)
    try:
        with N.Context(0, sz.I, sz.J, sz.K) as ctx:
            ctx.init_device()
            ctx.jacobi_device(nn, 1)
            used = N.last_two_step_kernel()
            p, g = ctx.read_field("p", 1), ctx.read_gosa(1)
    finally:
        lib.hp_set_temporal_blocking(old)
    if kernel == "tx":
        assert used == "k_stencil_tx"
    elif kernel == "tb2":
        assert used.startswith("k_stencil_tb2")
    assert np.array_equal(p, ref["fields"]["p"])
    assert abs(g - ref["gosa64"]) <= GOSA_RTOL * ref["gosa64"]


@pytest.mark.gpu
@pytest.mark.parametrize("env", [{"HIMENO_TB2_XS": "0"}, {"HIMENO_TB2_XS": "1"},
                                 {"HIMENO_TB2_STASH": "0"},
                                 {"HIMENO_TB2_XS": "0", "HIMENO_TB2_FLOW": "1"},
                                 {"HIMENO_TB2_XS": "1", "HIMENO_TB2_FLOW": "1"}])
@pytest.mark.parametrize("dims,nn", [((75, 45, 141), 6), ((129, 129, 257), 5)])
def test_two_step_stash_variants_bit_exact(gpu, monkeypatch, dims, nn, env):
    """Step-2 coefficients from the cross-warp stash (step-1 warps write the quads they
    loaded into tensor memory; default), from each step-2 warp's own copy, or straight
    from shared memory: the oracle's field bit for bit, per-pass and flow launches."""
    sz = himeno.custom_size(*dims)
    ref = oracle.run_program(sz.I, sz.J, sz.K, nn)
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    lib = N.load()
    old = lib.hp_set_temporal_blocking(1)
    try:
        with N.Context(0, sz.I, sz.J, sz.K) as ctx:
            ctx.init_device()
            ctx.jacobi_device(nn, 1)
            assert N.last_two_step_kernel().startswith("k_stencil_tb2")
            p, g = ctx.read_field("p", 1), ctx.read_gosa(1)
    finally:
        lib.hp_set_temporal_blocking(old)
    assert np.array_equal(p, ref["fields"]["p"])
    assert abs(g - ref["gosa64"]) <= GOSA_RTOL * ref["gosa64"]
