"""Velocity-slab decomposition of the uniform 1D+1V path.

Each slab owns all x and a contiguous range of nv / S velocity cells, stored as its own uniform
level (UniformVlasov1D with carried velocity ghosts and the fused field).  Per RK4 stage:

1. every slab runs its fused stage kernel: f_next, the slab's moment rho_j = base_j - dv sum f
   (base 1 on slab 0, 0 elsewhere, vlasov_level_set_moment_base), and the characteristic
   velocity ghosts of f_next at both slab faces;
2. the moments are summed over the slabs (all-reduce): rho = 1 - dv sum_v f on every slab, the
   input of the next stage's field (each slab evaluates the same E redundantly, as the paper
   keeps configuration space undistributed);
3. halo exchange: the two lowest / highest interior velocity columns of f_next
   (vlasov_vslab_pack) go to the lower / upper neighbour, which writes them into its ghost
   columns (vlasov_vslab_unpack) -- interior slab faces are not physical boundaries.

`comm` implements steps 2-3 over the slabs this process owns: DistComm (one slab per rank,
torch.distributed: NCCL all-reduce and send/recv; gloo for the CPU logic tests) or LocalComm
(all slabs in one process on one GPU, the single-GPU emulation the parity tests use).
"""
from __future__ import annotations

from typing import List, Optional, Sequence

import numpy as np
import torch

from . import api
from ._lib import CENTERED4
from .solver import UniformVlasov1D


def slab_ranges(nv: int, nslabs: int) -> List[range]:
    """Contiguous velocity ranges of the slabs; each a multiple of 4 cells (in-kernel ghost mode)."""
    if nv % (4 * nslabs):
        raise ValueError(f"nv = {nv} must be a multiple of 4 x the number of slabs ({nslabs})")
    n = nv // nslabs
    return [range(j * n, (j + 1) * n) for j in range(nslabs)]


class LocalComm:
    """All slabs in this process (one GPU): the sum and the neighbour copies run on the slabs'
    shared stream."""

    def allreduce(self, slabs, bufs):
        total = bufs[0].clone()
        for b in bufs[1:]:
            total += b
        for b in bufs:
            b.copy_(total)
        return []

    def exchange(self, slabs):
        n = len(slabs)
        for j, s in enumerate(slabs):
            if j > 0:
                s.lo_recv.copy_(slabs[j - 1].hi_send)
            if j < n - 1:
                s.hi_recv.copy_(slabs[j + 1].lo_send)
        return []


class DistComm:
    """One slab per rank (rank r owns slab r of `world`): torch.distributed collectives.

    Both transports are stream-ordered: with NCCL, torch runs each operation on the
    communicator's internal stream after an event on the caller's current stream, and
    `work.wait()` makes the caller's stream wait for it (the host does not block), so a whole
    step can be captured in one CUDA graph (VSlabVlasov1D.capture).  The moment all-reduce and
    the halo send/recv use two process groups (two NCCL communicators, two internal streams):
    the 16 KiB all-reduce and the 32 KiB neighbour exchange of a stage run concurrently."""

    def __init__(self, rank: int, world: int, group=None, p2p_group=None):
        import torch.distributed as dist
        self.dist = dist
        self.rank, self.world, self.group = rank, world, group
        self.p2p_group = p2p_group if p2p_group is not None else group

    @classmethod
    def with_p2p_group(cls, rank: int, world: int):
        """All ranks must call this together: a second communicator for the halo exchange."""
        import torch.distributed as dist
        return cls(rank, world, None, dist.new_group(list(range(world))))

    def allreduce(self, slabs, bufs):
        works = [self.dist.all_reduce(b, op=self.dist.ReduceOp.SUM, group=self.group, async_op=True) for b in bufs]
        return works

    def exchange(self, slabs):
        (s,) = slabs
        dist, r, n = self.dist, self.rank, self.world
        g = self.p2p_group
        ops = []
        if r > 0:
            ops.append(dist.P2POp(dist.isend, s.lo_send, r - 1, g))
            ops.append(dist.P2POp(dist.irecv, s.lo_recv, r - 1, g))
        if r < n - 1:
            ops.append(dist.P2POp(dist.isend, s.hi_send, r + 1, g))
            ops.append(dist.P2POp(dist.irecv, s.hi_recv, r + 1, g))
        return dist.batch_isend_irecv(ops) if ops else []


class _Slab:
    def __init__(self, j, nslabs, vr, w_ncells, lower, dx, f0v_full, recon, stream):
        self.j, self.nslabs, self.vr = j, nslabs, vr
        nvs = len(vr)
        lo_v = lower[1] + vr.start * dx[1]
        self.S = UniformVlasov1D((w_ncells[0], nvs), (lower[0], lo_v), dx, [((0, 0), (w_ncells[0] - 1, nvs - 1))],
                                 np.asarray(f0v_full)[vr.start:vr.start + nvs + 4], recon, stream=stream,
                                 fused=True, carry_ghosts=True)
        api.vlasov_level_set_moment_base(self.S.level.h, 1.0 if j == 0 else 0.0)
        api.vlasov_level_set_velocity_faces(self.S.level.h, j == 0, j == nslabs - 1)
        nx = w_ncells[0]
        with torch.cuda.stream(self.S.stream):
            z = lambda: torch.zeros(2 * nx, dtype=torch.float64, device="cuda")   # noqa: E731
            self.lo_send, self.hi_send, self.lo_recv, self.hi_recv = z(), z(), z(), z()

    @property
    def has_lo(self):
        return self.j > 0

    @property
    def has_hi(self):
        return self.j < self.nslabs - 1

    def pack(self, f):
        api.vlasov_vslab_pack(self.S.level.h, f, self.lo_send if self.has_lo else None,
                              self.hi_send if self.has_hi else None)

    def unpack(self, f):
        api.vlasov_vslab_unpack(self.S.level.h, f, self.lo_recv if self.has_lo else None,
                                self.hi_recv if self.has_hi else None)


class VSlabVlasov1D:
    """The slabs `owned` (indices into the nslabs velocity slabs) of a uniform 1D+1V problem.

    ncells, lower, dx, f0v_full: the whole problem (f0v_full on the ghosted global v range).
    LocalComm: owned = all slabs; DistComm: owned = [rank]."""

    def __init__(self, ncells: Sequence[int], lower, dx, f0v_full, nslabs: int, owned: Sequence[int], comm,
                 recon: int = CENTERED4, stream: Optional[torch.cuda.Stream] = None):
        self.ncells, self.lower, self.dx = tuple(ncells), tuple(lower), tuple(dx)
        self.nslabs = nslabs
        self.ranges = slab_ranges(ncells[1], nslabs)
        self.comm = comm
        self.stream = stream or torch.cuda.Stream()
        self.slabs = [_Slab(j, nslabs, self.ranges[j], ncells, lower, dx, f0v_full, recon, self.stream) for j in owned]

    # ------------------------------------------------------------------ state
    def set_state(self, f_full):
        """f_full: the whole nx x nv state (each slab takes its velocity range), or a callable
        vrange -> the nx x len(vrange) state of that velocity range (only the owned slabs)."""
        with torch.cuda.stream(self.stream):
            for s in self.slabs:
                S = s.S
                a = f_full(s.vr) if callable(f_full) else f_full[:, s.vr.start:s.vr.stop]
                S.level.set_domain(S.A, np.ascontiguousarray(a))
                api.vlasov_reduce_charge([S.level.h], [S.A], -1.0, 1.0 if s.j == 0 else 0.0, 0, S.rhos[0])
            for wk in self.comm.allreduce(self.slabs, [s.S.rhos[0] for s in self.slabs]):
                wk.wait()
            for s in self.slabs:
                S = s.S
                S.poisson.solve(S.rhos[0], None, S.E[0], 2)
                api.vlasov_fill_ghosts(S.level.h, S.A, None, None, S.E[0], S.f0v)
            self._halo(lambda S: S.A)
        self.stream.synchronize()

    def get_state(self) -> List[np.ndarray]:
        return [s.S.get_state() for s in self.slabs]

    def _halo(self, field_of, extra_works=()):
        for s in self.slabs:
            s.pack(field_of(s.S))
        works = list(extra_works) + list(self.comm.exchange(self.slabs))
        for w in works:                      # stream-ordered: the current stream waits, not the host
            w.wait()
        for s in self.slabs:
            s.unpack(field_of(s.S))

    # ------------------------------------------------------------------ step
    def stage(self, st: int, dt: float):
        for s in self.slabs:
            s.S.stage_launch(st, dt)
        rho_next = [(s.S.rhos[1] if st % 2 == 1 else s.S.rhos[0]) for s in self.slabs]
        # the moment all-reduce and the halo exchange are issued back to back (two communicators)
        # and waited for together before the next stage
        works = self.comm.allreduce(self.slabs, rho_next)
        self._halo(lambda S: S.buffers(st)[1], works)

    def step(self, dt: float):
        with torch.cuda.stream(self.stream):
            for st in (1, 2, 3, 4):
                self.stage(st, dt)

    def capture(self, dt: float):
        """One step as a CUDA graph (the stage kernels, pack / unpack and the NCCL operations);
        one eager step first (NCCL communicators and lazily built plans exist before capture)."""
        self.step(dt)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=self.stream):
            for st in (1, 2, 3, 4):
                self.stage(st, dt)
        self.graph = g
        return g

    def replay(self):
        with torch.cuda.stream(self.stream):
            self.graph.replay()
