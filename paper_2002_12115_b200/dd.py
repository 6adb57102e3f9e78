"""Slab decomposition of the device-resident Jacobi over several B200s.

Partition: the interior planes [1, I-2) of the slowest dimension (C ``i``; BASELINE
calls the configs "k-decomposed", but in the ``[i][j][k]`` layout k is contiguous and
splitting ``i`` gives the same 1-D topology with contiguous halo planes) are split into
contiguous, near-equal slabs of at least two planes.  Each slab carries two halo planes
per side; every pass runs one or two iterations (the two-step kernel's first step also
recomputes the neighbours' adjacent planes) and then exchanges two J x P planes of p with
each neighbour; the fp64 gosa partials are summed once at the end of the jacobi call (only
the last iteration's gosa is observable).  Device work and transfers run in the native library
(``csrc/decomp.cpp``):

* ``SlabJacobi``  one process per GPU (torchrun); halo planes and the gosa all-reduce
  over NCCL on the library stream, NCCL id broadcast through ``torch.distributed``;
* ``GroupJacobi`` one process driving several slabs (several GPUs, or several virtual
  ranks on one GPU -- how the decomposition is tested on a single device).
"""

from __future__ import annotations

from . import native as N
from .apps import himeno


HALO = N.SLAB_HALO    # halo planes per side


def slab_range(I: int, nranks: int, rank: int) -> tuple:
    """Interior planes [i_begin, i_end) owned by `rank` (same rule as hp_slab_range)."""
    n = I - 3
    if I < 4 or not 1 <= nranks <= n or not 0 <= rank < nranks or \
            (nranks > 1 and nranks > n // HALO):
        raise ValueError(f"cannot split {n} interior planes over {nranks} ranks (rank {rank})")
    return 1 + rank * n // nranks, 1 + (rank + 1) * n // nranks


def halo_plan(I: int, nranks: int) -> list:
    """(rank, sends, receives) after each pass: (peer, first local plane) of HALO planes.

    Rank r's local plane li is global plane i_begin-HALO+li: its first HALO interior
    planes (local HALO..) go to rank r-1's upper halo, its last HALO to rank r+1's lower
    halo (local 0..).  Mirrors hp_group_jacobi / hp_dd_jacobi.
    """
    out = []
    for r in range(nranks):
        b, e = slab_range(I, nranks, r)
        n = e - b
        sends, recvs = [], []
        if r > 0:
            sends.append((r - 1, HALO))
            recvs.append((r - 1, 0))
        if r < nranks - 1:
            sends.append((r + 1, n))
            recvs.append((r + 1, n + HALO))
        out.append((r, sends, recvs))
    return out


def group_nccl_id(rank: int, world: int, dist=None) -> bytes:
    """Rank 0 creates the NCCL unique id, every rank receives it (torch.distributed)."""
    if world <= 1:
        return b""
    if dist is None:
        import torch.distributed as dist  # noqa: F811
    obj = [N.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    return obj[0]


class SlabJacobi:
    """This rank's slab of a Himeno grid on one GPU; exchange over NCCL."""

    def __init__(self, size, rank: int, world: int, device: int, dist=None):
        self.size = himeno.size(size)
        self.rank, self.world = rank, world
        self.slab = slab_range(self.size.I, world, rank)
        sz = self.size
        self.ctx = N.Context(device, sz.I, sz.J, sz.K, slab=self.slab)
        self.ctx.dd_init(world, rank, group_nccl_id(rank, world, dist))
        self.ctx.init_device()

    @property
    def interior_points(self) -> int:
        b, e = self.slab
        return (e - b) * (self.size.J - 3) * (self.size.K - 3)

    def jacobi(self, nn: int) -> None:
        """Enqueue nn iterations (halo exchange after each) + the gosa all-reduce."""
        self.ctx.dd_jacobi(nn)

    def time_steps(self, steps: int, nn: int) -> float:
        return self.ctx.dd_time_steps(steps, nn)

    def gosa(self) -> float:
        return self.ctx.read_gosa(1)

    def interior_p(self):
        """This slab's interior planes of p (global planes [i_begin, i_end))."""
        return self.ctx.read_field("p", 1)[HALO:-HALO]

    def close(self) -> None:
        self.ctx.close()


class GroupJacobi:
    """Several slabs driven by one process (devices may repeat: virtual ranks)."""

    def __init__(self, size, devices):
        self.size = himeno.size(size)
        sz = self.size
        n = len(devices)
        self.slabs = [slab_range(sz.I, n, r) for r in range(n)]
        self.contexts = [N.Context(d, sz.I, sz.J, sz.K, slab=s)
                         for d, s in zip(devices, self.slabs)]
        for c in self.contexts:
            c.init_device()

    def jacobi(self, nn: int) -> float:
        return N.group_jacobi(self.contexts, nn)

    def gather(self, name: str = "p"):
        """The full I x J x K field: slab interiors + the global boundary planes."""
        import numpy as np
        sz = self.size
        out = np.zeros((sz.I, sz.J, sz.K), dtype=np.float32)
        for c, (b, e) in zip(self.contexts, self.slabs):
            local = c.read_field(name, 1)
            out[b:e] = local[HALO:-HALO]
            if b == 1:
                out[0] = local[HALO - 1]
            if e == sz.I - 2:
                out[e] = local[-HALO]
        return out

    def close(self) -> None:
        for c in self.contexts:
            c.close()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()
