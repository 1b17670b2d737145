"""Step orchestration for a single uniform level (1D+1V Vlasov-Poisson), issuing only libvlasov
C-ABI calls on one CUDA stream (optionally captured in a CUDA graph).

One RK4 step = Alg.5 with one hierarchy and one level, per stage s = 1..4:
    vlasov_reduce_moment (fused partials of the previous stage)      rho
    vlasov_poisson_solve                                             E
    vlasov_inject_field                                              E_lvl
    vlasov_fill_ghosts(f_s, E_bc = E of the previous evaluation)      (Alg.2; reading #6b)
    vlasov_rk4_stage(s)  -> f_{s+1} and its per-tile partial sums    (Alg.3 + P:389-410)
Buffers: A = f_n, B = f2/f4, C = f3, U = u.  E_lvl alternates between two buffers so that the
ghost fill of stage s reads the field of stage s-1 while stage s uses its own.
"""
from __future__ import annotations

from typing import Optional, Sequence

import numpy as np
import torch

from . import api
from ._lib import CENTERED4


class UniformVlasov1D:
    def __init__(self, ncells: Sequence[int], lower: Sequence[float], dx: Sequence[float], boxes,
                 f0v: np.ndarray, recon: int = CENTERED4, stream: Optional[torch.cuda.Stream] = None):
        self.stream = stream or torch.cuda.Stream()
        self.ncells = tuple(ncells)
        self.dx = tuple(dx)
        self.recon = recon
        with torch.cuda.stream(self.stream):
            self.level = api.Level(2, ncells, lower, dx, (1, 1), boxes, stream=self.stream)
            info = self.level.info
            if info.partial_doubles == 0:
                raise ValueError("UniformVlasov1D needs boxes that tile the domain")
            self.poisson = api.Poisson(ncells[0], dx[0], self.stream)
            self.A = self.level.field()
            self.B = self.level.field()
            self.C = self.level.field()
            self.U = self.level.field()
            self.E = [self.level.efield(), self.level.efield()]
            self.rho = torch.zeros(ncells[0], dtype=torch.float64, device="cuda")
            self.Efin = torch.zeros(ncells[0], dtype=torch.float64, device="cuda")
            self.partials = torch.zeros(info.partial_doubles, dtype=torch.float64, device="cuda")
            self.f0v = torch.as_tensor(np.ascontiguousarray(f0v), dtype=torch.float64).cuda()
        self.graph = None
        self.graph_steps = 0
        self.dt = None

    # ------------------------------------------------------------------ state
    def set_state(self, f_full: np.ndarray):
        with torch.cuda.stream(self.stream):
            self.level.set_domain(self.A, f_full)
            # first constraint evaluation (t = 0): direct moment of f_n
            api.vlasov_reduce_moment([self.level.h], [self.A], None, self.rho)
            self._field(self.E[0])
        self.stream.synchronize()

    def get_state(self) -> np.ndarray:
        self.stream.synchronize()
        return self.level.get_domain(self.A)

    def field_state(self) -> np.ndarray:
        """E of the last constraint evaluation (interior, level resolution)."""
        self.stream.synchronize()
        return self.E[0][2:-2].cpu().numpy()

    # ------------------------------------------------------------------ step
    def _field(self, E_out):
        self.poisson.solve(self.rho, None, self.Efin)
        api.vlasov_inject_field(self.level.h, self.Efin, (self.ncells[0],), E_out)

    def _stage(self, s, dt):
        L = self.level.h
        A, B, C, U = self.A, self.B, self.C, self.U
        f_s, f_next = {1: (A, B), 2: (B, C), 3: (C, B), 4: (B, A)}[s]
        E_cur, E_bc = (self.E[1], self.E[0]) if s % 2 == 1 else (self.E[0], self.E[1])
        if s > 1 or self._have_partials:
            api.vlasov_reduce_moment([L], None, self.partials, self.rho)
        else:
            api.vlasov_reduce_moment([L], [A], None, self.rho)
        self._field(E_cur)
        api.vlasov_fill_ghosts(L, f_s, None, None, E_bc, self.f0v)
        api.vlasov_rk4_stage(L, s, dt, A, f_s, U, f_next, E_cur, self.recon, self.partials)

    def step(self, dt: float):
        with torch.cuda.stream(self.stream):
            for s in (1, 2, 3, 4):
                self._stage(s, dt)
        self._have_partials = True

    _have_partials = False

    def capture(self, dt: float, steps: int = 1):
        """Capture `steps` RK4 steps (16*steps... launches) in a CUDA graph."""
        self.step(dt)                         # warm-up (also makes fused partials available)
        self.stream.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=self.stream):
            for _ in range(steps):
                for s in (1, 2, 3, 4):
                    self._stage(s, dt)
        self.graph, self.graph_steps, self.dt = g, steps, dt
        return g

    def replay(self):
        with torch.cuda.stream(self.stream):
            self.graph.replay()

    def launches_per_step(self) -> int:
        # per stage: sum_partials, circulant(E), inject, fill(copy+phys = 2), stage
        return 4 * 6
