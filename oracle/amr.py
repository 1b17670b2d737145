"""Oracle: multi-level block-structured AMR advance for 1D+1V.  TEST INFRASTRUCTURE ONLY.

Follows PAPER.md section 3 step by step:
  Alg.1/5  synchronous RK4 over all levels with one dt
  Alg.2    predictor state: f_pred = f_old + alpha_s dt k; interpolate fine ghosts from the
           coarser level; exchange ghosts; physical boundary condition
           (reading #15: level by level coarse -> fine; within a level siblings, then CF,
           then PHYS)
  Alg.3    fluxes on every patch of every level, F_accum += b_s F
  Alg.4    update finest -> coarsest from accumulated fluxes, coarse faces under fine faces
           take the mean of the fine F* (reading #14), then average down f_new
  constraints: Alg.8 sub-patch reduction -> rho on the finest x mesh -> Poisson -> E ->
           injection to every level
  regrid: tags delta1 + delta2 > tol, dilation by the tag buffer, fixed-tile
           boxes (reading #18); new fine patches copy old fine data where they overlap, else
           interpolate from the coarse level.
"""
from __future__ import annotations

import numpy as np

from . import boxes, field, interp, reduction, scheme, uniform

G = 2
RK_ALPHA, RK_B = uniform.RK_ALPHA, uniform.RK_B


class Hierarchy:
    """1D+1V phase-space hierarchy: geometry, level metadata and ghosted patch data."""

    def __init__(self, lower, h0, ncells0, level_boxes, ratios, fbg_fn, recon=scheme.CENTERED4,
                 interp_mode=interp.LINEAR5):
        """level_boxes[l]: boxes in level-l index space; ratios[l]: ratio of level l to level 0;
        fbg_fn(ratio) -> unperturbed profile on the ghosted v range of that level."""
        self.lower = tuple(lower)
        self.h0 = tuple(h0)
        self.ncells0 = tuple(ncells0)
        self.domain0 = boxes.box((0, 0), (ncells0[0] - 1, ncells0[1] - 1))
        self.periodic = (True, False)
        self.recon = recon
        self.interp_mode = interp_mode
        self.fbg_fn = fbg_fn
        self.set_levels(level_boxes, ratios)

    def set_levels(self, level_boxes, ratios):
        self.levels = [boxes.LevelMeta(self.domain0, r, bl, self.periodic)
                       for bl, r in zip(level_boxes, ratios)]
        self.fbg = [self.fbg_fn(l.ratio) for l in self.levels]
        self.maps = []
        for l, lvl in enumerate(self.levels):
            coarser = self.levels[l - 1] if l > 0 else None
            if coarser is not None and not boxes.properly_nested(lvl, coarser):
                raise ValueError(f"level {l} not nested")
            self.maps.append([boxes.ghost_map(lvl, p, coarser) for p in range(len(lvl.boxes))])

    def h(self, l):
        r = self.levels[l].ratio
        return (self.h0[0] / r[0], self.h0[1] / r[1])

    def nx_finest(self):
        return self.ncells0[0] * self.levels[-1].ratio[0]

    def new_data(self):
        return [[np.full(tuple(s + 2 * G for s in boxes.size(b)), np.nan) for b in lvl.boxes]
                for lvl in self.levels]

    def cells(self):
        return sum(boxes.ncells(b) for lvl in self.levels for b in lvl.boxes)


# --------------------------------------------------------------------------- ghosts
def _interior(a):
    return a[G:-G, G:-G]


def fill_ghosts(H, data, E_bc_levels):
    """Alg.2 ghost fill of every level, coarse -> fine, in place."""
    for l, lvl in enumerate(H.levels):
        coarse = H.levels[l - 1] if l > 0 else None
        rr = None if coarse is None else tuple(f // c for f, c in zip(lvl.ratio, coarse.ratio))
        for p, b in enumerate(lvl.boxes):
            kind, sp, sc = H.maps[l][p]
            fg = data[l][p]
            gb = boxes.grow(b, G)
            phys = []
            for t, c in enumerate(boxes.cells_of(gb)):
                li, lj = c[0] - gb[0][0], c[1] - gb[0][1]
                if kind[t] == boxes.SIBLING:
                    qb = lvl.boxes[sp[t]]
                    w = lvl.wrap(c)
                    fg[li, lj] = data[l][sp[t]][w[0] - qb[0][0] + G, w[1] - qb[0][1] + G]
                elif kind[t] == boxes.COARSE:
                    w = lvl.wrap(c)
                    cc = (w[0] // rr[0], w[1] // rr[1])
                    cb = coarse.boxes[sp[t]]
                    cg = data[l - 1][sp[t]]
                    ci, cj = cc[0] - cb[0][0] + G, cc[1] - cb[0][1] + G
                    block = cg[ci - 2: ci + 3, cj - 2: cj + 3]
                    fg[li, lj] = interp.interp_fine_cell_2d(
                        block, rr[0], rr[1], w[0] - cc[0] * rr[0], w[1] - cc[1] * rr[1], H.interp_mode)
                elif kind[t] == boxes.PHYS:
                    phys.append((li, lj, c))
            # physical v boundary last (needs the x-ghost columns), reading #6
            E_l = E_bc_levels[l]
            nvd = lvl.domain[1][1] + 1
            for li, lj, c in phys:
                a = -E_l[lvl.wrap(c)[0]]
                fbg = H.fbg[l]
                if c[1] < 0:
                    f0, f1, f2, f3 = (fg[li, lj + (-c[1]) + m] for m in range(4))  # cells j=0..3
                    g1, g2 = uniform.extrapolate_low(f0, f1, f2, f3)
                    val = (g1 if c[1] == -1 else g2) if a < 0 else fbg[c[1] + G]
                else:
                    off = c[1] - (nvd - 1)                                      # 1 or 2
                    f0, f1, f2, f3 = (fg[li, lj - off - m] for m in range(4))   # cells n-1..n-4
                    g1, g2 = uniform.extrapolate_low(f0, f1, f2, f3)
                    val = (g1 if off == 1 else g2) if a > 0 else fbg[c[1] + G]
                fg[li, lj] = val


# --------------------------------------------------------------------------- constraints
def constraints(H, data):
    """Sub-patch reduction -> periodic Poisson on the finest x mesh -> E_finest -> E per level."""
    rho = reduction.subpatch_reduce(H.levels, data, H.h0[1], H.ncells0[0])
    dxf = H.h0[0] / H.levels[-1].ratio[0]
    E_f = field.efield_from_rho(rho, dxf)
    rxf = H.levels[-1].ratio[0]
    return [reduction.inject(E_f, rxf // lvl.ratio[0]) for lvl in H.levels], rho


def patch_rhs(H, l, p, fg, E_l):
    b = H.levels[l].boxes[p]
    hx, hv = H.h(l)
    vb = scheme.exact_vbar(H.lower[1] + b[0][1] * hv, hv, boxes.size(b)[1])
    Eg = field.ghost_periodic(E_l)
    Ep = Eg[b[0][0]: b[1][0] + 2 * G + 1]
    return scheme.rhs(fg, [vb], [Ep], (hx, hv), H.recon)


# --------------------------------------------------------------------------- update
def coarsen_fluxes_into(H, l, F_fine_lvl, F_coarse_lvl):
    """Alg.4 "coarsen fluxes down to level l-1": every coarse face that coincides with a face
    of a level-l patch takes the mean of the overlying fine F* (reading #14)."""
    fine, coarse = H.levels[l], H.levels[l - 1]
    rx, rv = (f // c for f, c in zip(fine.ratio, coarse.ratio))
    ncx = coarse.domain[1][0] + 1
    for q, fb in enumerate(fine.boxes):
        Fx, Fv = F_fine_lvl[q]
        fx0, fv0 = fb[0]
        nfx, nfv = boxes.size(fb)
        for p, cb in enumerate(coarse.boxes):
            Cx, Cv = F_coarse_lvl[p]
            # x-faces: fine face index a (0..nfx) is at fine position fx0 + a - 1/2
            for a in range(nfx + 1):
                xf = fx0 + a                         # fine cell to the right of the face
                if xf % rx:
                    continue
                for xc in (xf // rx, xf // rx - ncx, xf // rx + ncx):   # periodic images
                    for jc in range(fv0 // rv, (fv0 + nfv) // rv):
                        ia, ja = xc - cb[0][0], jc - cb[0][1]
                        if 0 <= ia <= cb[1][0] - cb[0][0] + 1 and 0 <= ja <= cb[1][1] - cb[0][1]:
                            rows = [jc * rv + s - fv0 for s in range(rv)]
                            Cx[ia, ja] = np.mean([Fx[a, r] for r in rows])
            # v-faces: fine face index m (0..nfv) is at fine position fv0 + m - 1/2
            for m in range(nfv + 1):
                vf = fv0 + m
                if vf % rv:
                    continue
                vc = vf // rv
                for ic in range(fx0 // rx, (fx0 + nfx) // rx):
                    ia, ja = ic - cb[0][0], vc - cb[0][1]
                    if 0 <= ia <= cb[1][0] - cb[0][0] and 0 <= ja <= cb[1][1] - cb[0][1] + 1:
                        cols = [ic * rx + s - fx0 for s in range(rx)]
                        Cv[ia, ja] = np.mean([Fv[c, m] for c in cols])


def average_down(H, data):
    """Coarse cells under a finer patch := mean of the fine cell averages (reading
    #14), finest -> coarsest, in place on the interiors."""
    for l in range(len(H.levels) - 1, 0, -1):
        fine, coarse = H.levels[l], H.levels[l - 1]
        rx, rv = (f // c for f, c in zip(fine.ratio, coarse.ratio))
        for q, fb in enumerate(fine.boxes):
            ff = _interior(data[l][q])
            cbox = boxes.coarsen(fb, (rx, rv))
            mean = ff.reshape(ff.shape[0] // rx, rx, ff.shape[1] // rv, rv).mean(axis=(1, 3))
            for p, cb in enumerate(coarse.boxes):
                ov = boxes.intersect(cb, cbox)
                if boxes.is_empty(ov):
                    continue
                cf = _interior(data[l - 1][p])
                cf[ov[0][0] - cb[0][0]: ov[1][0] - cb[0][0] + 1, ov[0][1] - cb[0][1]: ov[1][1] - cb[0][1] + 1] = \
                    mean[ov[0][0] - cbox[0][0]: ov[1][0] - cbox[0][0] + 1, ov[0][1] - cbox[0][1]: ov[1][1] - cbox[0][1] + 1]


def end_of_step_constraints(H, data, E_bc):
    """Alg.5's ComputeInstantaneousConstraints(f_new) after ComputeUpdate: ghosts of
    f_new (with the latest field E_bc for the boundary condition, reading #6b), then the
    constraints.  Its E is the boundary-condition field of the next step's stage 1."""
    fill_ghosts(H, data, E_bc)
    E_new, _ = constraints(H, data)
    return E_new


def step(H, data, E_bc, dt):
    """One synchronous RK4 step (Alg.5, one hierarchy).  ``data`` holds f_old (interiors);
    E_bc: per-level E of the previous constraint evaluation, E(f_old) (reading #6b).
    Returns (new data, E(f_new) = the end-of-step constraint evaluation, flux ledger of F*)."""
    L = len(H.levels)
    f_old = [[_interior(a).copy() for a in lvl] for lvl in data]
    k = [[np.zeros_like(a) for a in lvl] for lvl in f_old]
    F_acc = [[None] * len(lvl.boxes) for lvl in H.levels]
    for s in range(4):
        pred = H.new_data()
        for l in range(L):                                                 # Alg.2
            for p in range(len(H.levels[l].boxes)):
                _interior(pred[l][p])[...] = f_old[l][p] + RK_ALPHA[s] * dt * k[l][p]
        fill_ghosts(H, pred, E_bc)
        E_lv, _ = constraints(H, pred)                                      # Alg.5
        for l in range(L):                                                 # Alg.3
            for p in range(len(H.levels[l].boxes)):
                k[l][p], F = patch_rhs(H, l, p, pred[l][p], E_lv[l])
                F_acc[l][p] = [RK_B[s] * Fd for Fd in F] if F_acc[l][p] is None else \
                    [Fa + RK_B[s] * Fd for Fa, Fd in zip(F_acc[l][p], F)]
        E_bc = E_lv
    new = H.new_data()
    for l in range(L - 1, -1, -1):                                         # Alg.4
        if l + 1 < L:
            coarsen_fluxes_into(H, l + 1, F_acc[l + 1], F_acc[l])
        for p in range(len(H.levels[l].boxes)):
            _interior(new[l][p])[...] = f_old[l][p] + dt * scheme.divergence(F_acc[l][p], H.h(l))
    average_down(H, new)
    return new, end_of_step_constraints(H, new, E_bc), F_acc


# --------------------------------------------------------------------------- tags / regrid
def tag_cells(fg, hx, hv, tol):
    """delta1 f + delta2 f > tol on the interior of a ghosted 2D array, evaluated
    in this fixed order without contraction:
      d1 = sqrt(0.5 * (hx*(fx+ - fx-)^2 + hv*(fv+ - fv-)^2))
      d2 = 0.5 * (hx*hx*|fx+ - 2f + fx-| + hv*hv*|fv+ - 2f + fv-|)."""
    f = fg[G:-G, G:-G]
    xp, xm = fg[G + 1:fg.shape[0] - G + 1, G:-G], fg[G - 1:fg.shape[0] - G - 1, G:-G]
    vp, vm = fg[G:-G, G + 1:fg.shape[1] - G + 1], fg[G:-G, G - 1:fg.shape[1] - G - 1]
    dx1 = xp - xm
    dv1 = vp - vm
    d1 = np.sqrt(0.5 * (hx * (dx1 * dx1) + hv * (dv1 * dv1)))
    sx = (xp - 2.0 * f) + xm
    sv = (vp - 2.0 * f) + vm
    d2 = 0.5 * ((hx * hx) * np.abs(sx) + (hv * hv) * np.abs(sv))
    return (d1 + d2) > tol


def level0_tags(H, data, tol):
    """Tags over the whole level-0 domain (level 0 tiles the domain)."""
    lvl = H.levels[0]
    t = np.zeros(H.ncells0, dtype=bool)
    hx, hv = H.h(0)
    for p, b in enumerate(lvl.boxes):
        t[b[0][0]: b[1][0] + 1, b[0][1]: b[1][1] + 1] = tag_cells(data[0][p], hx, hv, tol)
    return t


def level_tags(H, data, l, tol):
    """Tags of level l's patches on its whole level domain (False off the patches);
    the level's ghosts must be filled."""
    lvl = H.levels[l]
    t = np.zeros(boxes.size(lvl.domain), dtype=bool)
    hx, hv = H.h(l)
    for p, b in enumerate(lvl.boxes):
        t[b[0][0]: b[1][0] + 1, b[0][1]: b[1][1] + 1] = tag_cells(data[l][p], hx, hv, tol)
    return t


def new_level_boxes(level, tags, ratio, smallest, largest, efficiency, nest=1):
    """Boxes of the next finer level from the (dilated) tags of `level` (reading #28): tags kept
    inside the nesting region of `level` (boxes.nesting_mask), clustered (clustering.cluster_tags
    in level cells; smallest / largest are finer-level patch sizes converted by the ratio), each
    cluster intersected with the nesting region (boxes.mask_to_boxes), refined by `ratio`."""
    from . import clustering
    nm = boxes.nesting_mask(level, nest)
    t = np.asarray(tags, bool) & nm
    sm = [-(-smallest[d] // ratio[d]) for d in range(2)]
    lg = [max(sm[d], largest[d] // ratio[d]) for d in range(2)]
    out = []
    for b in clustering.cluster_tags(t, sm, lg, efficiency):
        sub = nm[b[0][0]: b[1][0] + 1, b[0][1]: b[1][1] + 1]
        out.extend(boxes.mask_to_boxes(sub, b[0]))
    return boxes.sort_boxes([boxes.refine(b, ratio) for b in out])


def regrid_hierarchy(H, data, E_bc, tol, buffers, ratios, smallest, largest, efficiency=0.7):
    """Multi-level regrid: for k = 0, 1, ...: fill the ghosts of the new
    levels 0..k (E_bc kept for existing level indices, 0 for new ones), tag level k (buffer[k]),
    build level k+1 by new_level_boxes(ratio[k], smallest[k], largest[k]); its data copies the old
    level k+1 where they overlap, else is interpolated from the new level k.  Stops
    when a level has no tags or len(ratios) fine levels exist.  ratios[k]: ratio of level k+1 to k.
    Returns (new data, list of new boxes per fine level)."""
    old_levels, old_data = H.levels, data
    lb = [old_levels[0].boxes]
    rs = [old_levels[0].ratio]
    H.set_levels(lb, rs)
    new = [[a.copy() for a in old_data[0]]]
    out_boxes = []
    for k in range(len(ratios)):
        E_fill = [E_bc[l] if (l < len(old_levels) and old_levels[l].ratio == H.levels[l].ratio)
                  else np.zeros(H.ncells0[0] * H.levels[l].ratio[0]) for l in range(len(H.levels))]
        fill_ghosts(H, new, E_fill)
        tags = boxes.dilate_tags(level_tags(H, new, k, tol), buffers[k], (True, False))
        nb = new_level_boxes(H.levels[k], tags, ratios[k], smallest[k], largest[k], efficiency)
        if not nb:
            break
        r_next = tuple(a * b for a, b in zip(H.levels[k].ratio, ratios[k]))
        H.set_levels(lb + [nb], rs + [r_next])
        lb, rs = lb + [nb], rs + [r_next]
        fine_new = [np.full(tuple(n + 2 * G for n in boxes.size(b)), np.nan) for b in nb]
        rr = tuple(ratios[k])
        for q, b in enumerate(nb):
            fine = _interior(fine_new[q])
            for p, cb in enumerate(H.levels[k].boxes):          # interpolate from the new level k
                cbox = boxes.intersect(boxes.coarsen(b, rr), cb)
                if boxes.is_empty(cbox):
                    continue
                cg = new[k][p]
                sub = cg[cbox[0][0] - cb[0][0]: cbox[1][0] - cb[0][0] + 2 * G + 1,
                         cbox[0][1] - cb[0][1]: cbox[1][1] - cb[0][1] + 2 * G + 1]
                ref = interp.refine_patch_2d(sub, rr[0], rr[1], H.interp_mode)
                fb = boxes.refine(cbox, rr)
                fine[fb[0][0] - b[0][0]: fb[1][0] - b[0][0] + 1, fb[0][1] - b[0][1]: fb[1][1] - b[0][1] + 1] = ref
            if k + 1 < len(old_levels) and old_levels[k + 1].ratio == r_next:   # copy old level k+1
                for op, ob in enumerate(old_levels[k + 1].boxes):
                    ov = boxes.intersect(ob, b)
                    if boxes.is_empty(ov):
                        continue
                    fine[ov[0][0] - b[0][0]: ov[1][0] - b[0][0] + 1, ov[0][1] - b[0][1]: ov[1][1] - b[0][1] + 1] = \
                        _interior(old_data[k + 1][op])[ov[0][0] - ob[0][0]: ov[1][0] - ob[0][0] + 1,
                                                       ov[0][1] - ob[0][1]: ov[1][1] - ob[0][1] + 1]
        new.append(fine_new)
        out_boxes.append(nb)
    return new, out_boxes


def regrid_two_level(H, data, E_bc, tol, buffer, ratio, tile):
    """Tag level 0, dilate, tile -> new level-1 boxes; move data (copy old fine where the new
    patch overlaps it, else interpolate from level 0).  Level 0 ghosts must be filled.
    Returns (new data, new level-1 boxes)."""
    tags = boxes.dilate_tags(level0_tags(H, data, tol), buffer, (True, False))
    new_boxes = boxes.tiles_from_tags(tags, ratio, tile)
    return regrid_to(H, data, new_boxes, ratio), new_boxes


def regrid_two_level_clustered(H, data, E_bc, tol, buffer, ratio, smallest, largest, efficiency=0.7):
    """As regrid_two_level, with the level-1 boxes grouped from the dilated level-0 tags by
    clustering.cluster_tags (reading #28); smallest / largest are level-1 patch sizes
     in level-1 cells, converted to level-0 cells (ceil / floor by the ratio)."""
    from . import clustering
    tags = boxes.dilate_tags(level0_tags(H, data, tol), buffer, (True, False))
    sm = [-(-smallest[d] // ratio[d]) for d in range(2)]
    lg = [max(sm[d], largest[d] // ratio[d]) for d in range(2)]
    coarse = clustering.cluster_tags(tags, sm, lg, efficiency)
    new_boxes = boxes.sort_boxes([boxes.refine(b, ratio) for b in coarse])
    return regrid_to(H, data, new_boxes, ratio), new_boxes


def regrid_to(H, data, new_boxes, ratio):
    """Data motion of a two-level regrid to the level-1 boxes `new_boxes`: new fine
    patches copy old fine data where they overlap it, else are interpolated from level 0."""
    old_levels = H.levels
    old_data = data
    lb = [old_levels[0].boxes] + ([new_boxes] if new_boxes else [])
    rs = [old_levels[0].ratio] + ([tuple(ratio)] if new_boxes else [])
    H.set_levels(lb, rs)
    new = H.new_data()
    for p in range(len(H.levels[0].boxes)):
        new[0][p][...] = old_data[0][p]
    if new_boxes:
        for q, nb in enumerate(H.levels[1].boxes):
            fine = _interior(new[1][q])
            # interpolate everything from the coarse level first ...
            for p, cb in enumerate(H.levels[0].boxes):
                cbox = boxes.intersect(boxes.coarsen(nb, ratio), cb)
                if boxes.is_empty(cbox):
                    continue
                cg = old_data[0][p]
                sub = cg[cbox[0][0] - cb[0][0]: cbox[1][0] - cb[0][0] + 2 * G + 1,
                         cbox[0][1] - cb[0][1]: cbox[1][1] - cb[0][1] + 2 * G + 1]
                ref = interp.refine_patch_2d(sub, ratio[0], ratio[1], H.interp_mode)
                fb = boxes.refine(cbox, ratio)
                fine[fb[0][0] - nb[0][0]: fb[1][0] - nb[0][0] + 1, fb[0][1] - nb[0][1]: fb[1][1] - nb[0][1] + 1] = ref
            # ... then copy old fine data where it exists (same-level copy wins)
            if len(old_levels) > 1:
                for op, ob in enumerate(old_levels[1].boxes):
                    ov = boxes.intersect(ob, nb)
                    if boxes.is_empty(ov):
                        continue
                    fine[ov[0][0] - nb[0][0]: ov[1][0] - nb[0][0] + 1, ov[0][1] - nb[0][1]: ov[1][1] - nb[0][1] + 1] = \
                        _interior(old_data[1][op])[ov[0][0] - ob[0][0]: ov[1][0] - ob[0][0] + 1,
                                                   ov[0][1] - ob[0][1]: ov[1][1] - ob[0][1] + 1]
    return new
