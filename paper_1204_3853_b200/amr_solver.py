"""Step orchestration for a 1D+1V phase-space hierarchy (block-structured AMR), issuing only
libvlasov C-ABI calls on one CUDA stream.

One RK4 step = Alg.5 with one hierarchy, Alg.1-4 over the levels:

    zero the interface flux registers of every fine level
    for s = 1..4:                                   (f_s = f_n, f2, f3, f4 per level)
        vlasov_fill_ghosts  level 0 .. L-1          Alg.2: siblings / periodic, CF interpolation
                                                    from the (already filled) coarser level,
                                                    characteristic v-BC with E_bc (reading #6b)
        vlasov_reduce_moment                         Alg.8 sub-patch reduction -> rho (finest x)
        vlasov_poisson_solve                         P:283-311 -> E on the finest x mesh
        vlasov_inject_field per level
        vlasov_rk4_stage per level                   Alg.3: faces, fluxes, divergence, RK4 combine
        vlasov_flux_register_accumulate per fine level   += b_s (F_coarse - <F_fine>) on the
                                                    coarse-fine interface (Alg.3 F_accum)
    vlasov_average_down level L-1 .. 1              Alg.4: refluxing (flux substitution) and
                                                    coarse := mean of fine
    vlasov_fill_ghosts + constraints of f_new       Alg.5's ComputeInstantaneousConstraints(f_new)
                                                    (P:676-684): the E_bc of the next stage 1

Regrid (C3 rule, reading #18): tags on level 0, dilation, fixed fine tiles,
vlasov_level_fill_from (copy old fine where it overlaps, else interpolate from level 0), then a
constraint evaluation on the new hierarchy (Alg.5 after regridHierarchies).
"""
from __future__ import annotations

from typing import List, Optional, Sequence

import numpy as np
import torch

from . import api
from ._lib import CENTERED4, LINEAR5

RK_B = (1.0 / 6.0, 1.0 / 3.0, 1.0 / 3.0, 1.0 / 6.0)


class AmrVlasov1D:
    def __init__(self, ncells0: Sequence[int], lower: Sequence[float], dx0: Sequence[float], level_boxes,
                 ratios, f0v_fn, recon: int = CENTERED4, interp: int = LINEAR5,
                 stream: Optional[torch.cuda.Stream] = None):
        """level_boxes[l]: boxes (lo, hi) in level-l index space; ratios[l]: ratio to level 0;
        f0v_fn(ratio) -> unperturbed profile on the ghosted v range of a level (numpy)."""
        self.stream = stream or torch.cuda.Stream()
        self.ncells0 = tuple(ncells0)
        self.lower = tuple(lower)
        self.dx0 = tuple(dx0)
        self.recon = recon
        self.interp = interp
        self.f0v_fn = f0v_fn
        self.levels: List[api.Level] = []
        self.bufs = []            # per level: dict A, B, C, U
        self.E = []               # per level: [E_a, E_b] ghosted level fields
        self.f0v = []
        self.regs = []            # per level (None for level 0)
        self.cur = 0              # which of E[l][0/1] holds E_bc
        self._f0v_cache = {}
        with torch.cuda.stream(self.stream):
            for l, (bl, r) in enumerate(zip(level_boxes, ratios)):
                self._append_level(bl, r)
        self._make_field_plan()

    # ------------------------------------------------------------------ construction
    def _append_level(self, boxes, ratio):
        coarser = self.levels[-1] if self.levels else None
        L = api.Level(2, self.ncells0, self.lower, self.dx0, ratio, boxes, coarser=coarser, stream=self.stream)
        self.levels.append(L)
        self.bufs.append({k: L.field(0.0) for k in "ABCU"})
        self.E.append([L.efield(), L.efield()])
        key = tuple(ratio)
        if key not in self._f0v_cache:     # the unperturbed profile of a ratio (kept across regrids)
            self._f0v_cache[key] = torch.as_tensor(np.ascontiguousarray(self.f0v_fn(key)), dtype=torch.float64).cuda()
        self.f0v.append(self._f0v_cache[key])
        n = L.info.fluxreg_doubles
        self.regs.append(None if coarser is None else torch.zeros(max(1, n), dtype=torch.float64, device="cuda"))

    def _make_field_plan(self):
        nxf = self.levels[-1].info.domain_cells[0]
        dxf = self.dx0[0] / self.levels[-1].ratio[0]
        if getattr(self, "poisson", None) is not None and (nxf, dxf) == (self.nxf, self.dxf):
            return                          # same finest mesh after a regrid: keep the plan
        self.nxf, self.dxf = nxf, dxf
        self.poisson = api.Poisson(self.nxf, self.dxf, self.stream)
        self.rho = torch.zeros(self.nxf, dtype=torch.float64, device="cuda")
        self.E_f = torch.zeros(self.nxf, dtype=torch.float64, device="cuda")

    @property
    def handles(self):
        return [L.h for L in self.levels]

    # ------------------------------------------------------------------ state
    def set_state(self, level_arrays, constraints: bool = True):
        """level_arrays[l]: whole-level-domain array (only patch cells are read) or a list of
        per-patch interior arrays.  constraints=False: only load f (a multi-species driver then
        evaluates the joint constraints)."""
        with torch.cuda.stream(self.stream):
            for L, b, a in zip(self.levels, self.bufs, level_arrays):
                if isinstance(a, (list, tuple)):
                    L.set_patches(b["A"], a)
                else:
                    L.set_domain(b["A"], a)
            for E in self.E:
                E[0].zero_()
                E[1].zero_()
            self.cur = 0
            if constraints:
                self._initial_constraints()
        self.stream.synchronize()

    def _initial_constraints(self):
        """Ghosts with the current E_bc, then E_bc := constraints(f_n) (Alg.5 start / after regrid)."""
        A = [b["A"] for b in self.bufs]
        self._fill(A, [E[self.cur] for E in self.E])
        self._constraints(A, [E[self.cur] for E in self.E])

    def get_state(self, ghost=0):
        self.stream.synchronize()
        return [L.get_patches(b["A"], ghost) for L, b in zip(self.levels, self.bufs)]

    def field_state(self):
        self.stream.synchronize()
        return [E[self.cur][2:-2].cpu().numpy() for E in self.E]

    # ------------------------------------------------------------------ pieces
    def _fill(self, fs, E_bc):
        for l, L in enumerate(self.levels):
            cL = self.levels[l - 1].h if l else None
            api.vlasov_fill_ghosts(L.h, fs[l], cL, fs[l - 1] if l else None, E_bc[l], self.f0v[l], self.interp)

    def _constraints(self, fs, E_out):
        api.vlasov_reduce_moment(self.handles, fs, self.rho)
        # the finest level is at the finest x resolution: the solve writes its ghosted E directly
        # (ghost = 2, vlasov_poisson_solve), the coarser levels are injected from its interior
        E_fin = E_out[-1]
        self.poisson.solve(self.rho, None, E_fin, 2)
        for l in range(len(self.levels) - 1):
            api.vlasov_inject_field(self.levels[l].h, E_fin[2:], (self.nxf,), E_out[l])

    def _stage(self, s, dt):
        order = {1: ("A", "B"), 2: ("B", "C"), 3: ("C", "B"), 4: ("B", "A")}[s]
        fs = [b[order[0]] for b in self.bufs]
        fnext = [b[order[1]] for b in self.bufs]
        E_bc = [E[self.cur] for E in self.E]
        E_cur = [E[1 - self.cur] for E in self.E]
        self._fill(fs, E_bc)
        self._constraints(fs, E_cur)
        for l, L in enumerate(self.levels):
            b = self.bufs[l]
            api.vlasov_rk4_stage(L.h, s, dt, b["A"], fs[l], b["U"], fnext[l], E_cur[l], None, None, self.recon,
                                 None)
        for l in range(1, len(self.levels)):
            api.vlasov_flux_register_accumulate(self.levels[l].h, fs[l], E_cur[l], fs[l - 1], E_cur[l - 1],
                                                RK_B[s - 1], self.regs[l], self.recon)
        self.cur = 1 - self.cur

    def step(self, dt: float):
        with torch.cuda.stream(self.stream):
            self._step_launches(dt)

    def _step_launches(self, dt):
        for r in self.regs[1:]:
            r.zero_()
        for s in (1, 2, 3, 4):
            self._stage(s, dt)
        for l in range(len(self.levels) - 1, 0, -1):
            api.vlasov_average_down(self.levels[l].h, self.bufs[l]["A"], self.bufs[l - 1]["A"], self.regs[l], dt)
        self._initial_constraints()          # Alg.5: constraints(f_new), reading #6b

    def step_graph(self, dt: float):
        """One step through a CUDA graph of the step's launches (captured on first use for the
        current hierarchy and dt; an eager step first builds the lazily created reduction plan).
        The E_bc ping-pong index returns to its value after 4 stages, so the graph is reusable."""
        key = (tuple(L.h.value for L in self.levels), float(dt))
        if getattr(self, "_graph_key", None) != key:
            if getattr(self, "_graph_key", None) is None:
                # first capture: one eager step builds the lazily created plans (Alg.8 reduction);
                # after a regrid the constraint evaluation in regrid_to has built them already
                self.step(dt)
                self.stream.synchronize()
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=self.stream):
                    self._step_launches(dt)
                self._graph, self._graph_key = g, key
                return
            self.stream.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=self.stream):
                self._step_launches(dt)
            self._graph, self._graph_key = g, key
        with torch.cuda.stream(self.stream):
            self._graph.replay()

    def next_dt(self, dt_prev, cfl=0.5, growth=1.1):
        """Adaptive step (reading #29) from the last constraint evaluation: one C-ABI
        call (vlasov_next_dt; max|E_l| reduced on the device, the rate formed in the library)."""
        return api.vlasov_next_dt(self.handles, [E[self.cur] for E in self.E], dt_prev, cfl, growth)

    def launches_per_step(self) -> int:
        nl = len(self.levels)
        # per stage: fill (copy/CF + phys) per level, reduction (2), Poisson (1, into the finest
        # level's E), inject per coarser level, stage kernel per level, flux registers per fine
        # level; then refluxing + average-down and the end-of-step constraint evaluation
        return 4 * (2 * nl + 2 + 1 + (nl - 1) + nl + (nl - 1)) + 2 * (nl - 1) + (2 * nl + 2 + 1 + (nl - 1))

    # ------------------------------------------------------------------ regrid (C3 rule)
    def tags_level0(self, tol, buffer):
        L0 = self.levels[0]
        with torch.cuda.stream(self.stream):
            self._fill([b["A"] for b in self.bufs], [E[self.cur] for E in self.E])
            tags = torch.zeros(L0.info.tag_bytes, dtype=torch.uint8, device="cuda")
            api.vlasov_tag_cells(L0.h, self.bufs[0]["A"], tol, buffer, tags)
        self.stream.synchronize()
        return tags.cpu().numpy().reshape(self.ncells0)

    def regrid(self, tol, buffer, ratio, tile):
        """Two-level regrid, C3 fixed-tile rule (reading #18): returns the new fine boxes."""
        tags = self.tags_level0(tol, buffer)
        return self.regrid_to(api.vlasov_tags_to_boxes(tags, self.ncells0, ratio, tile), ratio)

    def regrid_clustered(self, tol, buffer, ratio, smallest, largest, efficiency=0.7):
        """Two-level regrid with the level-1 boxes grouped from the dilated level-0 tags by
        vlasov_cluster_tags (reading #28); smallest / largest are level-1 patch sizes
         in level-1 cells, converted to level-0 cells (ceil / floor by the ratio)."""
        tags = self.tags_level0(tol, buffer)
        # clustering with the level-1 patch sizes converted to level-0 cells, refinement by the ratio
        # and sorting: all in the library (level 0 covers the domain, so nesting restricts nothing)
        fine = api.vlasov_regrid_boxes(self.levels[0].h, tags, ratio, smallest, largest, efficiency)
        return self.regrid_to(fine, ratio)

    def tags_level(self, k, tol, buffer):
        """Dilated tags of level k on its level domain (ghosts of levels 0..k filled first)."""
        L = self.levels[k]
        with torch.cuda.stream(self.stream):
            self._fill([b["A"] for b in self.bufs], [E[self.cur] for E in self.E])
            tags = torch.zeros(L.info.tag_bytes, dtype=torch.uint8, device="cuda")
            api.vlasov_tag_cells(L.h, self.bufs[k]["A"], tol, buffer, tags)
        self.stream.synchronize()
        return tags.cpu().numpy().reshape(tuple(L.info.domain_cells[d] for d in range(2)))

    def regrid_hierarchy(self, tol, buffers, ratios, smallest, largest, efficiency=0.7):
        """Multi-level regrid: for k = 0, 1, ...: ghosts of the new levels 0..k, tags of
        level k (buffers[k]), next-level boxes by vlasov_regrid_boxes (nesting in level k, clustering
        with the level-(k+1) patch sizes smallest[k] / largest[k], ratio ratios[k]); the new level
        k+1 copies the old level k+1 where they overlap, else interpolates from the new level k
        (vlasov_level_fill_from).  E_bc kept for surviving level indices, 0 for new ones; then the
        constraints of the new hierarchy.  Returns the list of new fine-level box lists."""
        old_levels, old_bufs, old_E = self.levels[1:], self.bufs[1:], [E[self.cur] for E in self.E[1:]]
        with torch.cuda.stream(self.stream):
            del self.levels[1:], self.bufs[1:], self.E[1:], self.f0v[1:], self.regs[1:]
        out = []
        for k in range(len(ratios)):
            tags = self.tags_level(k, tol, buffers[k])
            nb = api.vlasov_regrid_boxes(self.levels[k].h, tags, ratios[k], smallest[k], largest[k], efficiency)
            if not nb:
                break
            r_next = tuple(a * b for a, b in zip(self.levels[k].ratio, ratios[k]))
            with torch.cuda.stream(self.stream):
                self._append_level(nb, r_next)
                old = old_levels[k] if k < len(old_levels) and tuple(old_levels[k].ratio) == r_next else None
                api.vlasov_level_fill_from(self.levels[k + 1].h, self.bufs[k + 1]["A"], old.h if old else None,
                                           old_bufs[k]["A"] if old else None, self.levels[k].h, self.bufs[k]["A"],
                                           self.interp)
                if k < len(old_E) and old is not None:
                    self.E[k + 1][self.cur].copy_(old_E[k])
                else:
                    self.E[k + 1][self.cur].zero_()
            out.append(nb)
        with torch.cuda.stream(self.stream):
            self._make_field_plan()
            self._initial_constraints()
        self.stream.synchronize()
        del old_levels, old_bufs, old_E
        return out

    def regrid_to(self, new_boxes, ratio):
        """Replace level 1 by `new_boxes` (data: copy old fine where it overlaps, else interpolate
        from level 0; then the constraints of the new hierarchy)."""
        old_boxes = self.levels[1].boxes if len(self.levels) > 1 else []
        if [tuple(map(tuple, b)) for b in new_boxes] == [tuple(map(tuple, b)) for b in old_boxes] and \
                (len(self.levels) == 1 or tuple(self.levels[1].ratio) == tuple(ratio)):
            # same hierarchy: data unchanged; Alg.5 still re-evaluates the constraints
            with torch.cuda.stream(self.stream):
                self._initial_constraints()
            return new_boxes
        nlev_old = len(self.levels)
        old_level = self.levels[1] if nlev_old > 1 else None
        old_A = self.bufs[1]["A"] if nlev_old > 1 else None
        old_E = [E[self.cur] for E in self.E]
        with torch.cuda.stream(self.stream):
            del self.levels[1:], self.bufs[1:], self.E[1:], self.f0v[1:], self.regs[1:]
            if new_boxes:
                self._append_level(new_boxes, ratio)
                api.vlasov_level_fill_from(self.levels[1].h, self.bufs[1]["A"], old_level.h if old_level else None,
                                           old_A, self.levels[0].h, self.bufs[0]["A"], self.interp)
            # keep E_bc of the surviving levels, zero for new ones
            self.E[0][self.cur].copy_(old_E[0])
            if len(self.levels) > 1:
                if nlev_old > 1:
                    self.E[1][self.cur].copy_(old_E[1])
                else:
                    self.E[1][self.cur].zero_()
            self._make_field_plan()
            self._initial_constraints()
        self.stream.synchronize()
        del old_level
        return new_boxes

    def cells(self):
        """Cells on all levels (cached per hierarchy: the per-step host cost stays O(1))."""
        key = tuple(L.h.value for L in self.levels)
        if getattr(self, "_cells_key", None) != key:
            self._cells = sum((hi[0] - lo[0] + 1) * (hi[1] - lo[1] + 1) for L in self.levels for lo, hi in L.boxes)
            self._cells_key = key
        return self._cells


class MultiSpeciesVlasov1D:
    """Several species, one 1D+1V hierarchy (AmrVlasov1D) each, coupled only through the
    configuration-space field and advanced synchronously (Alg.5).  Per
    stage: the ghosts of every species (with its own previous field), the charge density
    rho = rho_bg + sum_s q_s n_s (vlasov_reduce_charge, accumulated over species), one Poisson
    solve on the common finest x mesh, and A_s = -(q_s/m_s) E injected into every level of species
    s (vlasov_inject_field_scaled; electrons A = E), then the stage kernels and flux registers of
    every species; after stage 4 the refluxing / average-down of every hierarchy."""

    def __init__(self, hierarchies, charges, masses, rho_bg=0.0):
        self.sp = list(hierarchies)
        self.q = [float(q) for q in charges]
        self.m = [float(m) for m in masses]
        self.rho_bg = float(rho_bg)
        nxf = {h.nxf for h in self.sp}
        if len(nxf) != 1:
            raise ValueError("species hierarchies must share the finest configuration mesh")
        self.stream = self.sp[0].stream
        # every C-ABI call enqueues on its level's stream: the species exchange rho and E every
        # stage, so their hierarchies must be built on one stream (else the stages race)
        if any(h.stream != self.stream for h in self.sp):
            raise ValueError("species hierarchies must share one CUDA stream (AmrVlasov1D(..., stream=s))")
        h0 = self.sp[0]
        self.nxf, self.dxf = h0.nxf, h0.dxf
        self.poisson = api.Poisson(self.nxf, self.dxf, self.stream)
        self.rho = torch.zeros(self.nxf, dtype=torch.float64, device="cuda")
        self.E_f = torch.zeros(self.nxf, dtype=torch.float64, device="cuda")

    def _constraints(self, fs_all, E_out_all):
        for i, (h, fs) in enumerate(zip(self.sp, fs_all)):
            api.vlasov_reduce_charge(h.handles, fs, self.q[i], self.rho_bg, i > 0, self.rho)
        self.poisson.solve(self.rho, None, self.E_f, 0)
        for i, h in enumerate(self.sp):
            for l, L in enumerate(h.levels):
                api.vlasov_inject_field_scaled(L.h, self.E_f, (self.nxf,), -self.q[i] / self.m[i], E_out_all[i][l])

    def set_state(self, states):
        """states[s]: level arrays of species s (as AmrVlasov1D.set_state)."""
        for h, st in zip(self.sp, states):
            h.set_state(st, constraints=False)
        with torch.cuda.stream(self.stream):
            A = [[b["A"] for b in h.bufs] for h in self.sp]
            for h, fs in zip(self.sp, A):
                h._fill(fs, [E[h.cur] for E in h.E])
            self._constraints(A, [[E[h.cur] for E in h.E] for h in self.sp])
        self.stream.synchronize()

    def step(self, dt):
        order = {1: ("A", "B"), 2: ("B", "C"), 3: ("C", "B"), 4: ("B", "A")}
        with torch.cuda.stream(self.stream):
            for h in self.sp:
                for r in h.regs[1:]:
                    r.zero_()
            for s in (1, 2, 3, 4):
                fs_all = [[b[order[s][0]] for b in h.bufs] for h in self.sp]
                for h, fs in zip(self.sp, fs_all):
                    h._fill(fs, [E[h.cur] for E in h.E])
                E_cur = [[E[1 - h.cur] for E in h.E] for h in self.sp]
                self._constraints(fs_all, E_cur)
                for i, h in enumerate(self.sp):
                    fnext = [b[order[s][1]] for b in h.bufs]
                    for l, L in enumerate(h.levels):
                        b = h.bufs[l]
                        api.vlasov_rk4_stage(L.h, s, dt, b["A"], fs_all[i][l], b["U"], fnext[l], E_cur[i][l], None,
                                             None, h.recon, None)
                    for l in range(1, len(h.levels)):
                        api.vlasov_flux_register_accumulate(h.levels[l].h, fs_all[i][l], E_cur[i][l],
                                                            fs_all[i][l - 1], E_cur[i][l - 1], RK_B[s - 1],
                                                            h.regs[l], h.recon)
                    h.cur = 1 - h.cur
            for h in self.sp:
                for l in range(len(h.levels) - 1, 0, -1):
                    api.vlasov_average_down(h.levels[l].h, h.bufs[l]["A"], h.bufs[l - 1]["A"], h.regs[l], dt)
            # Alg.5: the joint constraints of f_new (the next stage 1's boundary field, reading #6b)
            A = [[b["A"] for b in h.bufs] for h in self.sp]
            for h, fs in zip(self.sp, A):
                h._fill(fs, [E[h.cur] for E in h.E])
            self._constraints(A, [[E[h.cur] for E in h.E] for h in self.sp])

    def get_state(self):
        return [h.get_state() for h in self.sp]
