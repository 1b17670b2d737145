"""Step orchestration for a 2D+2V phase-space hierarchy (NEXT row N3), issuing only libvlasov C-ABI
calls on one CUDA stream.

One RK4 step = Alg.5 with one hierarchy, Alg.1-4 over the levels in the paper's F*
form:

    for s = 1..4:                                   (f_s = f_n, f2, f3, f4 per level)
        vlasov_fill_ghosts  level 0 .. L-1          Alg.2 in 4D: siblings / periodic images, CF
                                                    interpolation x, y, v_x, v_y, velocity BC
                                                    with E_bc (reading #6b)
        vlasov_reduce_moment                         Alg.8 4D -> 2D sub-patch reduction -> rho
        vlasov_poisson2d_solve                       2D periodic field (reading #32) -> E
        vlasov_inject_field_ghosted per level
        vlasov_rk4_stage_fstar per level             Alg.3: fluxes, F* += b_s F, next predictor
    vlasov_fstar_coarsen  level L-1 .. 1            Alg.4: coarse faces under fine faces
    vlasov_fstar_update   every level               f_new = f_n + dt div F*
    vlasov_average_down   level L-1 .. 1
    vlasov_fill_ghosts + constraints of f_new       Alg.5's ComputeInstantaneousConstraints(f_new)
"""
from __future__ import annotations

from typing import List, Optional, Sequence

import numpy as np
import torch

from . import api
from ._lib import CENTERED4, LINEAR5


class AmrVlasov2D2V:
    def __init__(self, ncells0: Sequence[int], lower: Sequence[float], dx0: Sequence[float], level_boxes,
                 ratios, f0v_fn, recon: int = CENTERED4, interp: int = LINEAR5,
                 stream: Optional[torch.cuda.Stream] = None):
        """level_boxes[l]: 4D boxes (lo, hi) in level-l index space; ratios[l]: ratio to level 0;
        f0v_fn(ratio) -> unperturbed profile on the ghosted (v_x, v_y) range of a level (numpy)."""
        self.stream = stream or torch.cuda.Stream()
        self.ncells0, self.lower, self.dx0 = tuple(ncells0), tuple(lower), tuple(dx0)
        self.recon, self.interp = recon, interp
        self.levels: List[api.Level] = []
        self.bufs, self.E, self.f0v, self.F = [], [], [], []
        self.cur = 0
        with torch.cuda.stream(self.stream):
            for bl, r in zip(level_boxes, ratios):
                L = api.Level(4, self.ncells0, self.lower, self.dx0, r, bl,
                              coarser=self.levels[-1] if self.levels else None, stream=self.stream)
                self.levels.append(L)
                self.bufs.append({k: L.field(0.0) for k in "ABC"})
                self.E.append([L.efield(), L.efield()])
                self.f0v.append(torch.as_tensor(np.ascontiguousarray(f0v_fn(tuple(r))).ravel(),
                                                dtype=torch.float64).cuda())
                self.F.append(torch.zeros(max(1, api.vlasov_level_face_doubles(L.h)), dtype=torch.float64,
                                          device="cuda"))
            rf = self.levels[-1].ratio
            self.nxf, self.nyf = self.ncells0[0] * rf[0], self.ncells0[1] * rf[1]
            self.poisson = api.Poisson2D(self.nxf, self.nyf, dx0[0] / rf[0], dx0[1] / rf[1], self.stream)
            self.rho = torch.zeros(self.nxf * self.nyf, dtype=torch.float64, device="cuda")
            self.E_f = torch.zeros(2 * (self.nxf + 4) * (self.nyf + 4), dtype=torch.float64, device="cuda")
        self.stream.synchronize()

    @property
    def handles(self):
        return [L.h for L in self.levels]

    def set_state(self, level_arrays):
        """level_arrays[l]: list of per-patch interior arrays.  Ghosts with E = 0, then the first
        constraint evaluation (Alg.5 start)."""
        with torch.cuda.stream(self.stream):
            for L, b, a in zip(self.levels, self.bufs, level_arrays):
                L.set_patches(b["A"], a)
            for E in self.E:
                E[0].zero_()
                E[1].zero_()
            self.cur = 0
            self._end_constraints()
        self.stream.synchronize()

    def get_state(self, ghost=0):
        self.stream.synchronize()
        return [L.get_patches(b["A"], ghost) for L, b in zip(self.levels, self.bufs)]

    def field_state(self):
        self.stream.synchronize()
        out = []
        for L, E in zip(self.levels, self.E):
            nx, ny = L.info.domain_cells[0], L.info.domain_cells[1]
            out.append(E[self.cur].view(2, nx + 4, ny + 4)[:, 2:-2, 2:-2].cpu().numpy())
        return out

    # ------------------------------------------------------------------ pieces
    def _fill(self, fs, E_bc):
        for l, L in enumerate(self.levels):
            api.vlasov_fill_ghosts(L.h, fs[l], self.levels[l - 1].h if l else None, fs[l - 1] if l else None,
                                   E_bc[l], self.f0v[l], self.interp)

    def _constraints(self, fs, E_out):
        api.vlasov_reduce_moment(self.handles, fs, self.rho)
        self.poisson.solve(self.rho, self.E_f)
        for L, e in zip(self.levels, E_out):
            api.vlasov_inject_field_ghosted(L.h, self.E_f, (self.nxf, self.nyf), e)

    def _end_constraints(self):
        """Ghosts with the current E_bc, then E_bc := constraints(f_n) (Alg.5 start / end of step)."""
        A = [b["A"] for b in self.bufs]
        self._fill(A, [E[self.cur] for E in self.E])
        self._constraints(A, [E[self.cur] for E in self.E])

    def step(self, dt: float):
        order = {1: ("A", "B"), 2: ("B", "C"), 3: ("C", "B"), 4: ("B", None)}
        with torch.cuda.stream(self.stream):
            for s in (1, 2, 3, 4):
                src, dst = order[s]
                fs = [b[src] for b in self.bufs]
                E_bc = [E[self.cur] for E in self.E]
                E_cur = [E[1 - self.cur] for E in self.E]
                self._fill(fs, E_bc)
                self._constraints(fs, E_cur)
                for l, L in enumerate(self.levels):
                    b = self.bufs[l]
                    api.vlasov_rk4_stage_fstar(L.h, s, dt, b["A"], fs[l], b[dst] if dst else None, E_cur[l],
                                               self.recon, self.F[l])
                self.cur = 1 - self.cur
            for l in range(len(self.levels) - 1, 0, -1):                # Alg.4, finest first
                api.vlasov_fstar_coarsen(self.levels[l].h, self.F[l], self.levels[l - 1].h, self.F[l - 1])
            for L, b, F in zip(self.levels, self.bufs, self.F):
                api.vlasov_fstar_update(L.h, dt, b["A"], F, b["A"])
            for l in range(len(self.levels) - 1, 0, -1):
                api.vlasov_average_down(self.levels[l].h, self.bufs[l]["A"], self.bufs[l - 1]["A"], None, dt)
            self._end_constraints()

    def cells(self):
        return sum(int(np.prod([hi[d] - lo[d] + 1 for d in range(4)])) for L in self.levels for lo, hi in L.boxes)
