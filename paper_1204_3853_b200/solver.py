"""Step orchestration for a single uniform level (1D+1V Vlasov-Poisson), issuing only libvlasov
C-ABI calls on one CUDA stream (optionally captured in a CUDA graph).

One RK4 step = Alg.5 with one hierarchy and one level.  Per stage s = 1..4:
    vlasov_poisson_solve(rho_s -> E_s, 2 periodic ghosts)          (injection at the
                                                                    finest x resolution is the
                                                                    identity)
    vlasov_rk4_stage(s, f_s, E_s, E_bc = E_{s-1})  -> f_{s+1}, rho_{s+1}
        (ghosts of f_s derived in-kernel = Alg.2 exchange + BC with the latest field, reading #6b:
         E_{s-1} for s >= 2, and for s = 1 E(f_n) = E_1 -- the end-of-step constraint evaluation
         of Alg.5, which on one periodic level is the stage-1 field itself;
         face averages, fluxes, divergence, RK4 combine P:233-410; moment P:295-297)
With ``self_ghost=False`` the ghost frame is filled by vlasov_fill_ghosts instead (generic path).
Buffers: A = f_n, B = f2/f4, C = f3, U = u.  E alternates between two buffers so that stage s
reads E_{s-1} for the boundary condition while it uses E_s for the fluxes.
"""
from __future__ import annotations

from typing import Optional, Sequence

import numpy as np
import torch

from . import api
from ._lib import CENTERED4


class UniformVlasov1D:
    def __init__(self, ncells: Sequence[int], lower: Sequence[float], dx: Sequence[float], boxes,
                 f0v: np.ndarray, recon: int = CENTERED4, stream: Optional[torch.cuda.Stream] = None,
                 self_ghost: bool = True, fused: Optional[bool] = None, carry_ghosts: bool = True):
        self.stream = stream or torch.cuda.Stream()
        self.ncells = tuple(ncells)
        self.dx = tuple(dx)
        self.recon = recon
        self.self_ghost = self_ghost
        # fused: constraint evaluation (Poisson + E) inside the stage kernel (vlasov_rk4_stage_vp)
        self.fused = (self_ghost and ncells[0] <= 4096 and ncells[0] % 2 == 0 and ncells[1] % 4 == 0) \
            if fused is None else fused
        # carry_ghosts (in-kernel ghost modes): every stage writes the velocity ghost columns of its
        # output for its own field (the next stage's E_bc), so stages read them instead of deriving
        # them from E_bc; set_state fills them once
        self.carry = self_ghost and carry_ghosts
        with torch.cuda.stream(self.stream):
            self.level = api.Level(2, ncells, lower, dx, (1, 1), boxes, stream=self.stream)
            if self.level.info.nblocks != 1:
                raise ValueError("UniformVlasov1D needs boxes that tile the domain")
            self.poisson = api.Poisson(ncells[0], dx[0], self.stream)
            self.A = self.level.field()
            self.B = self.level.field()
            self.C = self.level.field()
            self.U = self.level.field()
            self.E = [self.level.efield(), self.level.efield()]
            self.rhos = [torch.zeros(ncells[0], dtype=torch.float64, device="cuda") for _ in range(2)]
            self.rho = self.rhos[0]
            self.f0v = torch.as_tensor(np.ascontiguousarray(f0v), dtype=torch.float64).cuda()
        self.graph = None
        self.dt = None

    # ------------------------------------------------------------------ state
    def set_state(self, f_full: np.ndarray):
        with torch.cuda.stream(self.stream):
            self.level.set_domain(self.A, f_full)
            # first constraint evaluation (t = 0): moment of f_n, field -> E_bc of stage 1
            api.vlasov_reduce_moment([self.level.h], [self.A], self.rho)
            self.poisson.solve(self.rho, None, self.E[0], 2)
            # ghost frame of f_n for E(f_n) (stage 1 derives its own velocity ghosts; this is for the
            # other consumers of the state's ghosts, e.g. vlasov_reduce_current)
            api.vlasov_fill_ghosts(self.level.h, self.A, None, None, self.E[0], self.f0v)
        self.stream.synchronize()

    def get_state(self) -> np.ndarray:
        self.stream.synchronize()
        return self.level.get_domain(self.A)

    def field_state(self) -> np.ndarray:
        """E of the last constraint evaluation (interior, level resolution)."""
        self.stream.synchronize()
        return self.E[0][2:-2].cpu().numpy()

    # ------------------------------------------------------------------ step
    def buffers(self, s):
        A, B, C = self.A, self.B, self.C
        f_s, f_next = {1: (A, B), 2: (B, C), 3: (C, B), 4: (B, A)}[s]
        E_cur, E_bc = (self.E[1], self.E[0]) if s % 2 == 1 else (self.E[0], self.E[1])
        return f_s, f_next, E_cur, E_bc

    def field_launch(self, s):
        if self.fused:
            return                                  # inside the stage kernel
        _, _, E_cur, _ = self.buffers(s)
        self.poisson.solve(self.rho, None, E_cur, 2)

    def stage_launch(self, s, dt):
        L = self.level.h
        f_s, f_next, E_cur, E_bc = self.buffers(s)
        if self.fused:
            # rho ping-pong: stage s reads the moment of f_s and writes the moment of f_next
            rho_s, rho_n = (self.rhos[0], self.rhos[1]) if s % 2 == 1 else (self.rhos[1], self.rhos[0])
            api.vlasov_rk4_stage_vp(L, self.poisson.h, s, dt, self.A, f_s, self.U, f_next, rho_s, E_cur,
                                    None if self.carry else E_bc, self.f0v, self.recon, rho_n)
        elif self.self_ghost:
            api.vlasov_rk4_stage(L, s, dt, self.A, f_s, self.U, f_next, E_cur, None if self.carry else E_bc,
                                 self.f0v, self.recon, self.rho)
        else:
            # stage 1: the boundary field is E(f_n) = this stage's field (reading #6b)
            api.vlasov_fill_ghosts(L, f_s, None, None, E_cur if s == 1 else E_bc, self.f0v)
            api.vlasov_rk4_stage(L, s, dt, self.A, f_s, self.U, f_next, E_cur, None, None, self.recon, self.rho)

    def _stage(self, s, dt):
        self.field_launch(s)
        self.stage_launch(s, dt)

    def step(self, dt: float):
        with torch.cuda.stream(self.stream):
            for s in (1, 2, 3, 4):
                self._stage(s, dt)

    def capture(self, dt: float, steps: int = 1):
        """Warm up one step, then capture `steps` RK4 steps in a CUDA graph."""
        self.step(dt)
        self.stream.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=self.stream):
            for _ in range(steps):
                for s in (1, 2, 3, 4):
                    self._stage(s, dt)
        self.graph, self.dt = g, dt
        return g

    def replay(self):
        with torch.cuda.stream(self.stream):
            self.graph.replay()

    def launches_per_step(self) -> int:
        # per stage: fused stage kernel (with the field solve when fused; else + circulant)
        # (+ 2 ghost-fill kernels with stored ghosts)
        if self.fused:
            return 4
        return 4 * (2 if self.self_ghost else 4)


class UniformVlasov2D:
    """Uniform 2D+2V level.  field="prescribed" (BASELINE.json C5): a prescribed configuration-space
    field E(x, y) injected from a 2D mesh, its own previous constraint evaluation, so
    E_bc = E.  field="poisson" (N3, C5P): the self-consistent field of the 2D periodic Poisson
    problem (reading #32), re-evaluated at every predictor state (Alg.5).
    Per stage s = 1..4: the velocity ghost frame of f_s (characteristic condition with E_bc:
    E_{s-1}, or E(f_n) = E_1 at s = 1, reading #6b), one fused stage kernel whose epilogue writes
    per-(vx line, vy tile) moment partials, a tiny kernel summing them in a fixed order into
    rho(x, y) (the 4D -> 2D reduction, P:295-297 / P:1061-1072), and with field="poisson" the 2D
    field solve E(f_{s+1}) = -grad phi(rho) (vlasov_poisson2d_solve)."""

    def __init__(self, ncells, lower, dx, boxes, f0v: np.ndarray, E_mesh: Optional[np.ndarray] = None,
                 recon: int = CENTERED4, stream: Optional[torch.cuda.Stream] = None, field: str = "prescribed"):
        self.stream = stream or torch.cuda.Stream()
        self.ncells = tuple(ncells)
        self.recon = recon
        self.field = field
        if field not in ("prescribed", "poisson"):
            raise ValueError(field)
        with torch.cuda.stream(self.stream):
            self.level = api.Level(4, ncells, lower, dx, (1, 1, 1, 1), boxes, stream=self.stream)
            if self.level.info.nblocks != 1:
                raise ValueError("UniformVlasov2D needs boxes that tile the domain")
            self.A = self.level.field()
            self.B = self.level.field()
            self.C = self.level.field()
            self.U = self.level.field()
            self.rho = torch.zeros(ncells[0] * ncells[1], dtype=torch.float64, device="cuda")
            self.f0v = torch.as_tensor(np.ascontiguousarray(f0v), dtype=torch.float64).cuda()
            if field == "prescribed":
                self.E = self.level.efield()
                Em = torch.as_tensor(np.ascontiguousarray(E_mesh), dtype=torch.float64).cuda()
                api.vlasov_inject_field(self.level.h, Em, E_mesh.shape[1:], self.E)
            else:
                self.poisson = api.Poisson2D(ncells[0], ncells[1], dx[0], dx[1], self.stream)
                self.Es = [self.level.efield(), self.level.efield()]
                self.cur = 0                       # Es[cur] holds E(f_s) of the next stage
        self.stream.synchronize()
        self.graph = None

    def set_state(self, f_full: np.ndarray):
        with torch.cuda.stream(self.stream):
            self.level.set_domain(self.A, f_full)
            api.vlasov_reduce_moment([self.level.h], [self.A], self.rho)
            if self.field == "poisson":
                self.cur = 0
                self.poisson.solve(self.rho, self.Es[0])       # E(f_0), the first evaluation (Alg.5)
        self.stream.synchronize()

    def get_state(self) -> np.ndarray:
        self.stream.synchronize()
        return self.level.get_domain(self.A)

    def moment(self) -> np.ndarray:
        self.stream.synchronize()
        return self.rho.cpu().numpy().reshape(self.ncells[0], self.ncells[1])

    def field_state(self) -> np.ndarray:
        """E(f_n) (field="poisson"): (2, nx, ny) interior values of the last constraint evaluation."""
        self.stream.synchronize()
        nx, ny = self.ncells[:2]
        return self.Es[self.cur].view(2, nx + 4, ny + 4)[:, 2:-2, 2:-2].cpu().numpy()

    def stage_launch(self, s, dt):
        A, B, C = self.A, self.B, self.C
        f_s, f_next = {1: (A, B), 2: (B, C), 3: (C, B), 4: (B, A)}[s]
        if self.field == "prescribed":
            E, E_bc = self.E, self.E
        else:
            E = self.Es[self.cur]
            E_bc = E if s == 1 else self.Es[1 - self.cur]  # stage 1: E(f_n) (reading #6b)
        api.vlasov_rk4_stage(self.level.h, s, dt, A, f_s, self.U, f_next, E, E_bc, self.f0v, self.recon, self.rho)

    def field_launch(self, s):
        if self.field == "poisson":                        # E(f_{s+1}) from the fused moment
            self.poisson.solve(self.rho, self.Es[1 - self.cur])
            self.cur = 1 - self.cur

    def _stage(self, s, dt):
        self.stage_launch(s, dt)
        self.field_launch(s)

    def step(self, dt: float):
        with torch.cuda.stream(self.stream):
            for s in (1, 2, 3, 4):
                self._stage(s, dt)

    def capture(self, dt: float, steps: int = 1):
        self.step(dt)
        self.stream.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=self.stream):
            for _ in range(steps):
                for s in (1, 2, 3, 4):
                    self._stage(s, dt)
        self.graph, self.dt = g, dt
        return g

    def replay(self):
        with torch.cuda.stream(self.stream):
            self.graph.replay()

    def launches_per_step(self) -> int:
        # velocity ghost frame + stage kernel + moment finish (+ 2D field solve) per stage
        return 4 * (3 if self.field == "prescribed" else 4)
