"""Slab decomposition: partition/halo logic on CPU (gloo, world_size 2-3) and on GPU.

The CPU test runs the decomposition with host slabs: each gloo rank applies the
stencil to its slab in numpy float32 (every op rounds like the C program), swaps
halo planes with its neighbours exactly as hp_dd_jacobi does (dd.halo_plan), and
all-reduces the fp64 gosa; the gathered field must equal the full-grid oracle.
"""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle
from paper_2002_12115_b200 import dd
from paper_2002_12115_b200 import native as N
from paper_2002_12115_b200.apps import himeno

F32 = np.float32


def stencil_slab(f, lo, hi, jmax, kmax, omega=F32(0.8)):
    """Interior planes [lo, hi) of a slab (numpy float32, C evaluation order)."""
    p = f["p"]
    I_, J_, K_ = p.shape
    i, j, k = slice(lo, hi), slice(1, jmax - 1), slice(1, kmax - 1)

    def P(di, dj, dk):
        return p[lo + di:hi + di, 1 + dj:jmax - 1 + dj, 1 + dk:kmax - 1 + dk]

    c = (i, j, k)
    s0 = f["a0"][c] * P(1, 0, 0) + f["a1"][c] * P(0, 1, 0) + f["a2"][c] * P(0, 0, 1) \
        + f["b0"][c] * (P(1, 1, 0) - P(1, -1, 0) - P(-1, 1, 0) + P(-1, -1, 0)) \
        + f["b1"][c] * (P(0, 1, 1) - P(0, -1, 1) - P(0, 1, -1) + P(0, -1, -1)) \
        + f["b2"][c] * (P(1, 0, 1) - P(-1, 0, 1) - P(1, 0, -1) + P(-1, 0, -1)) \
        + f["c0"][c] * P(-1, 0, 0) + f["c1"][c] * P(0, -1, 0) + f["c2"][c] * P(0, 0, -1) \
        + f["wrk1"][c]
    ss = (s0 * f["a3"][c] - P(0, 0, 0)) * f["bnd"][c]
    out = p.copy()
    out[c] = P(0, 0, 0) + omega * ss
    assert out.dtype == F32
    return out, float(np.sum((ss * ss).astype(np.float64)))


def stencil_into(out, f, lo, hi, jmax, kmax, omega=F32(0.8)):
    """stencil_slab for planes [lo, hi) written into `out` (the overlapped schedule
    computes a slab's boundary planes and its interior in two calls)."""
    if hi <= lo:
        return 0.0
    new, part = stencil_slab(f, lo, hi, jmax, kmax, omega)
    out[lo:hi] = new[lo:hi]
    return part


def _rank_main(rank, world, name, nn, port, q, overlap=False):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sz = himeno.size(name)
    full = oracle.empty_fields(sz.I, sz.J, sz.K)
    oracle.initmt(full)
    b, e = dd.slab_range(sz.I, world, rank)
    H = dd.HALO
    lo = b - H                          # global plane of local plane 0 (may be -1)
    f = {}
    for k, v in full.items():
        pad = np.zeros((e - b + 2 * H,) + v.shape[1:], dtype=np.float32)
        src_lo, src_hi = max(lo, 0), min(e + H, v.shape[0])
        pad[src_lo - lo:src_hi - lo] = v[src_lo:src_hi]
        f[k] = pad
    plan = {r: (s, rv) for r, s, rv in dd.halo_plan(sz.I, world)}
    n = e - b
    gosa = 0.0
    for _ in range(nn):
        sends, recvs = plan[rank]
        if overlap and n >= 2 * H + 2:
            # hp_dd_jacobi's overlapped pass: the planes the neighbours need first,
            # their exchange in flight while the interior is computed, then the wait
            out = f["p"].copy()
            part = stencil_into(out, f, H, H + H, sz.J - 1, sz.K - 1)
            part += stencil_into(out, f, n, n + H, sz.J - 1, sz.K - 1)
            reqs = [dist.isend(torch.from_numpy(np.ascontiguousarray(out[pl:pl + H])), dst)
                    for dst, pl in sends]
            bufs = [(torch.empty(out[pl:pl + H].shape, dtype=torch.float32), src, pl)
                    for src, pl in recvs]
            reqs += [dist.irecv(buf, src) for buf, src, _ in bufs]
            part += stencil_into(out, f, H + H, n, sz.J - 1, sz.K - 1)   # the interior
            for r in reqs:
                r.wait()
            for buf, _, pl in bufs:
                out[pl:pl + H] = buf.numpy()
            f["p"] = out
        else:
            f["p"], part = stencil_slab(f, H, n + H, sz.J - 1, sz.K - 1)
            reqs = [dist.isend(torch.from_numpy(np.ascontiguousarray(f["p"][pl:pl + H])), dst)
                    for dst, pl in sends]
            for src, pl in recvs:
                buf = torch.empty(f["p"][pl:pl + H].shape, dtype=torch.float32)
                dist.recv(buf, src)
                f["p"][pl:pl + H] = buf.numpy()
            for r in reqs:
                r.wait()
        t = torch.tensor([part], dtype=torch.float64)
        dist.all_reduce(t)
        gosa = float(t.item())
    pieces = [None] * world
    dist.all_gather_object(pieces, (b, e, f["p"][H:-H]))
    if rank == 0:
        p = full["p"].copy()
        for bb, ee, arr in pieces:
            p[bb:ee] = arr
        ref = oracle.run_program(sz.I, sz.J, sz.K, nn)
        q.put((bool(np.array_equal(p, ref["fields"]["p"])), gosa, ref["gosa64"]))
    dist.destroy_process_group()


@pytest.mark.parametrize("overlap", [False, True])
@pytest.mark.parametrize("world", [2, 3])
def test_gloo_slab_decomposition_matches_oracle(world, overlap):
    """Host slabs with HALO-deep halos, exchanged per dd.halo_plan after every step --
    or, as hp_dd_jacobi overlaps it, boundary planes first, the exchange in flight
    (isend/irecv) while the interior is computed."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + world * 7 + int(overlap) * 3 + os.getpid() % 1000
    name = "XS" if overlap else "XXS"    # XS slabs are deep enough to split
    procs = [ctx.Process(target=_rank_main, args=(r, world, name, 3, port, q, overlap))
             for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    same, gosa, want = q.get(timeout=10)
    assert same
    assert abs(gosa - want) <= 1e-12 * want


def test_slab_range_partition():
    for I in (9, 33, 65, 257, 513):
        for n in range(1, min(9, (I - 3) // dd.HALO) + 1):
            ranges = [dd.slab_range(I, n, r) for r in range(n)]
            assert ranges[0][0] == 1 and ranges[-1][1] == I - 2
            assert all(a[1] == b[0] for a, b in zip(ranges, ranges[1:]))
            sizes = [e - b for b, e in ranges]
            assert max(sizes) - min(sizes) <= 1
            assert ranges == [N.slab_range(I, n, r) for r in range(n)]   # C ABI agrees
    with pytest.raises(ValueError):
        dd.slab_range(9, 7, 0)
    with pytest.raises(ValueError):
        dd.slab_range(9, 4, 0)          # 6 interior planes cannot give 4 slabs of >= 2


def test_halo_plan_is_symmetric():
    for world in (2, 3, 8):
        plan = dd.halo_plan(257, world)
        sends = {(r, dst) for r, s, _ in plan for dst, _ in s}
        recvs = {(src, r) for r, _, rv in plan for src, _ in rv}
        assert sends == recvs


@pytest.mark.gpu
@pytest.mark.parametrize("overlap", [0, 1])
@pytest.mark.parametrize("tb", [0, 1])
@pytest.mark.parametrize("ranks", [1, 2, 3, 4])
@pytest.mark.parametrize("name,nn", [("XS", 3), ("XS", 4), ("M", 2), ("M", 5)])
def test_gpu_group_slabs_match_oracle(gpu, monkeypatch, ranks, name, nn, tb, overlap):
    """Virtual ranks on one GPU, one- and two-step passes, halo exchange after each whole
    pass or overlapped with the interior (boundary planes first): bit-exact with the full
    grid."""
    monkeypatch.setenv("HIMENO_DD_OVERLAP", str(overlap))
    sz = himeno.size(name)
    ref = oracle.run_program(sz.I, sz.J, sz.K, nn)
    lib = N.load()
    old = lib.hp_set_temporal_blocking(tb)
    try:
        with dd.GroupJacobi(name, [0] * ranks) as g:
            gosa = g.jacobi(nn)
            p = g.gather("p")
    finally:
        lib.hp_set_temporal_blocking(old)
    assert np.array_equal(p, ref["fields"]["p"])
    assert abs(gosa - ref["gosa64"]) <= 1e-12 * ref["gosa64"]


@pytest.mark.gpu
def test_gpu_slab_single_rank_dd(gpu):
    """hp_dd_* with world 1 (no NCCL): same result as the full grid."""
    sz = himeno.size("XS")
    ref = oracle.run_program(sz.I, sz.J, sz.K, 3)
    s = dd.SlabJacobi("XS", 0, 1, 0)
    s.jacobi(3)
    assert abs(s.gosa() - ref["gosa64"]) <= 1e-12 * ref["gosa64"]
    assert np.array_equal(s.interior_p(), ref["fields"]["p"][1:sz.I - 2])
    s.jacobi(0)
    s.close()


@pytest.mark.gpu
def test_gpu_slab_single_rank_over_nccl(gpu):
    """hp_dd_* with a one-rank NCCL communicator: libnccl dlopen, ncclCommInitRank and the
    gosa ncclAllReduce run on the device (the halo send/recv needs a second GPU)."""
    sz = himeno.size("XS")
    ref = oracle.run_program(sz.I, sz.J, sz.K, 3)
    try:
        uid = N.nccl_unique_id()
    except Exception as exc:
        pytest.skip(f"NCCL unavailable: {exc}")
    s = dd.SlabJacobi("XS", 0, 1, 0)
    s.ctx.dd_init(1, 0, uid)
    s.ctx.init_device()
    s.jacobi(3)
    assert abs(s.gosa() - ref["gosa64"]) <= 1e-12 * ref["gosa64"]
    assert np.array_equal(s.interior_p(), ref["fields"]["p"][1:sz.I - 2])
    s.close()


def _id_main(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    uid = dd.group_nccl_id(rank, world, dist)
    ids = [None] * world
    dist.all_gather_object(ids, uid)
    if rank == 0:
        q.put(ids)
    dist.destroy_process_group()


def test_nccl_id_broadcast_over_gloo():
    """The NCCL id rank 0 creates (libnccl dlopen'ed by the library) reaches every rank."""
    try:
        N.nccl_unique_id()
    except Exception as exc:      # no libnccl in this environment
        pytest.skip(f"NCCL unavailable: {exc}")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29800 + os.getpid() % 1000
    procs = [ctx.Process(target=_id_main, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    ids = q.get(timeout=10)
    assert len(ids[0]) == 128 and ids[0] == ids[1]
