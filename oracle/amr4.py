"""Oracle: 2D+2V block-structured AMR (NEXT row N3).  TEST INFRASTRUCTURE ONLY.

The 1D+1V hierarchy oracle (amr.py) generalised to phase space (x, y, v_x, v_y) the way the paper
states its algorithms -- for arbitrary dimension (P:1000-1038 box calculus, P:1061-1072 the
reduction "elements 0 through N-1 configuration, N through N+M-1 velocity", "these
algorithms are applicable ... for arbitrary dimension"), here N = M = 2:

* ghost fill (Alg.2; reading #15 order): per level coarse -> fine, per patch
  siblings (after the periodic wrap of x and y), then coarse-fine interpolation from the parent
  coarse patch's ghosted data dimension by dimension x, y, v_x, v_y with linear5
  (default) or WENO5, then the characteristic velocity condition (reading #6) along
  v_x over the whole ghosted extent, then along v_y (the velocity corners take the v_y pass, as
  in the uniform oracle); a = -E_d of the cell's (x, y) column;
* constraints: Alg.8 Sub-Patch Reduction 4D -> 2D: sub-patches by Alg.7 (boxes.
  compute_sub_patches, reduction dims v_x, v_y), grown by 2 cells in x and y (reading #16),
  summed over both velocity dims including those ghost cells, the 2D partial sums refined in x
  then y to the finest configuration resolution, accumulated; the Alg.6 Mask Reduction as the
  comparator; rho -> the 2D periodic Poisson solve (field2d, reading #32) -> E = (E_x, E_y) ->
  injection per level (mean over the R_x x R_y finest cells);
* RHS per patch (scheme.rhs, the 4D operator), F* accumulation (Alg.3), Alg.4 flux coarsening
  (coarse faces under fine faces take the mean of the fine F* over the 3 transverse dims, reading
  #14) and average-down, the end-of-step constraint evaluation (Alg.5, reading #6b).
"""
from __future__ import annotations

import itertools

import numpy as np

from . import boxes, field, field2d, interp, scheme, uniform

G = 2
NDIM = 4
RK_ALPHA, RK_B = uniform.RK_ALPHA, uniform.RK_B


class Hierarchy4:
    def __init__(self, lower, h0, ncells0, level_boxes, ratios, fbg_fn, recon=scheme.CENTERED4,
                 interp_mode=interp.LINEAR5):
        """level_boxes[l]: 4D boxes in level-l index space; ratios[l]: ratio to level 0 per dim;
        fbg_fn(ratio) -> unperturbed profile on the ghosted (v_x, v_y) range of that level."""
        self.lower = tuple(float(x) for x in lower)
        self.h0 = tuple(float(x) for x in h0)
        self.ncells0 = tuple(int(n) for n in ncells0)
        self.domain0 = boxes.box((0,) * NDIM, tuple(n - 1 for n in ncells0))
        self.periodic = (True, True, False, False)
        self.recon = recon
        self.interp_mode = interp_mode
        self.fbg_fn = fbg_fn
        self.set_levels(level_boxes, ratios)

    def set_levels(self, level_boxes, ratios):
        self.levels = [boxes.LevelMeta(self.domain0, r, bl, self.periodic) for bl, r in zip(level_boxes, ratios)]
        self.fbg = [np.asarray(self.fbg_fn(tuple(l.ratio)), dtype=np.float64) for l in self.levels]
        for l in range(1, len(self.levels)):
            if not boxes.properly_nested(self.levels[l], self.levels[l - 1]):
                raise ValueError(f"level {l} not nested")

    def h(self, l):
        r = self.levels[l].ratio
        return tuple(self.h0[d] / r[d] for d in range(NDIM))

    def ncfg_finest(self):
        r = self.levels[-1].ratio
        return self.ncells0[0] * r[0], self.ncells0[1] * r[1]

    def new_data(self):
        return [[np.full(tuple(s + 2 * G for s in boxes.size(b)), np.nan) for b in lvl.boxes] for lvl in self.levels]

    def cells(self):
        return sum(boxes.ncells(b) for lvl in self.levels for b in lvl.boxes)


def _interior(a):
    return a[(slice(G, -G),) * NDIM]


def _sl(b, origin):
    """Slices of box b in an array whose element 0 sits at index `origin`."""
    return tuple(slice(b[0][d] - origin[d], b[1][d] - origin[d] + 1) for d in range(len(b[0])))


def _shift(b, s):
    return boxes.box([l + x for l, x in zip(b[0], s)], [h + x for h, x in zip(b[1], s)])


def _images(lvl):
    """Periodic shifts of the configuration dims (index space of the level)."""
    nx = lvl.domain[1][0] + 1
    ny = lvl.domain[1][1] + 1
    return [(sx, sy, 0, 0) for sx in (0, -nx, nx) for sy in (0, -ny, ny)]


# --------------------------------------------------------------------------- interpolation
def refine_patch_4d(cg, R, mode):
    """Refine every interior coarse cell of a ghosted (G = 2) 4D array: fine array (R_d n_d), one
    dimension at a time in the order x, y, v_x, v_y; each pass refines the interior
    coarse indices of its dimension on the (partly refined) array, the later dimensions still
    carrying their ghost cells."""
    a = np.asarray(cg, dtype=np.float64)
    for d in range(NDIM):
        n = a.shape[d] - 2 * G
        u5 = np.stack([np.take(a, np.arange(G - 2 + k, G - 2 + k + n), axis=d) for k in range(5)], axis=-1)
        fine = interp.interp_1d(u5, R[d], mode)                  # (..., n at axis d, ..., R_d)
        fine = np.moveaxis(fine, -1, d + 1)                      # (..., n, R_d, ...)
        shp = list(a.shape)
        shp[d] = n * R[d]
        a = fine.reshape(shp)              # dimension d refined (no ghost cells left along it)
    return a


def _refine_2d_interior(tg, Rx, Ry):
    """linear5 refinement of ghosted (G = 2) 2D partial sums, x then y: (Rx n_x, Ry n_y)."""
    nx, ny = tg.shape[0] - 2 * G, tg.shape[1] - 2 * G
    u5 = np.stack([tg[k: k + nx, :] for k in range(5)], axis=-1)
    xp = np.transpose(interp.linear5_1d(u5, Rx), (0, 2, 1)).reshape(nx * Rx, ny + 2 * G)
    v5 = np.stack([xp[:, k: k + ny] for k in range(5)], axis=-1)
    return interp.linear5_1d(v5, Ry).reshape(nx * Rx, ny * Ry)


# --------------------------------------------------------------------------- ghosts
def _apply_velocity_bc(fg, b, lvl, vd, E_l, fbg):
    """Characteristic condition along velocity dim vd (2 or 3) on the ghost layers of patch box b
    that lie outside the velocity domain, over the whole ghosted extent of the other dims."""
    comp = vd - 2
    gb = boxes.grow(b, G)
    Eg = field.ghost_periodic(E_l[comp])                     # level field with periodic ghosts
    a = -Eg[b[0][0]: b[1][0] + 2 * G + 1, b[0][1]: b[1][1] + 2 * G + 1]   # (x, y) of the ghosted box
    a = a[:, :, None, None]
    # profile on the patch's ghosted velocity range (fbg covers the level's ghosted range)
    prof = fbg[gb[0][2] + G: gb[1][2] + G + 1, gb[0][3] + G: gb[1][3] + G + 1][None, None, :, :]

    def take(j):                                              # ghosted index j along vd
        idx = [slice(None)] * NDIM
        idx[vd] = slice(j, j + 1)
        return tuple(idx)
    n = b[1][vd] - b[0][vd] + 1
    if 0 < b[0][vd] - lvl.domain[0][vd] < G or 0 < lvl.domain[1][vd] - b[1][vd] < G:
        raise ValueError("a patch must touch the velocity boundary or stay >= 2 cells from it")
    if b[0][vd] == lvl.domain[0][vd]:                         # low velocity boundary
        g1, g2 = uniform.extrapolate_low(fg[take(G)], fg[take(G + 1)], fg[take(G + 2)], fg[take(G + 3)])
        out = a < 0
        fg[take(G - 1)] = np.where(out, g1, prof[take(G - 1)])
        fg[take(G - 2)] = np.where(out, g2, prof[take(G - 2)])
    if b[1][vd] == lvl.domain[1][vd]:                         # high velocity boundary
        e = G + n - 1
        g1, g2 = uniform.extrapolate_low(fg[take(e)], fg[take(e - 1)], fg[take(e - 2)], fg[take(e - 3)])
        out = a > 0
        fg[take(e + 1)] = np.where(out, g1, prof[take(e + 1)])
        fg[take(e + 2)] = np.where(out, g2, prof[take(e + 2)])


def fill_ghosts(H, data, E_bc):
    """Alg.2 ghost fill of every level, coarse -> fine, in place.  E_bc[l]: (2, nx_l, ny_l)."""
    for l, lvl in enumerate(H.levels):
        coarse = H.levels[l - 1] if l > 0 else None
        rr = None if coarse is None else tuple(f // c for f, c in zip(lvl.ratio, coarse.ratio))
        vbox = boxes.box((-10 ** 9, -10 ** 9, lvl.domain[0][2], lvl.domain[0][3]),
                         (10 ** 9, 10 ** 9, lvl.domain[1][2], lvl.domain[1][3]))
        refined = {}                                          # coarse patch -> refined interior
        for p, b in enumerate(lvl.boxes):
            fg = data[l][p]
            gb = boxes.grow(b, G)
            filled = np.zeros(fg.shape, dtype=bool)
            filled[_sl(b, gb[0])] = True
            # (i) siblings and periodic images (same level)
            for q, qb in enumerate(lvl.boxes):
                for s in _images(lvl):
                    if q == p and s == (0, 0, 0, 0):
                        continue
                    reg = boxes.intersect(boxes.intersect(gb, _shift(qb, s)), vbox)
                    if boxes.is_empty(reg):
                        continue
                    src = _shift(reg, tuple(-x for x in s))
                    fg[_sl(reg, gb[0])] = data[l][q][_sl(src, boxes.grow(qb, G)[0])]
                    filled[_sl(reg, gb[0])] = True
            # (ii) coarse-fine interpolation from the parent coarse patch
            need = ~filled
            need &= _vmask(fg.shape, gb, lvl)
            if need.any():
                if coarse is None:
                    raise ValueError(f"level 0 patch {p} has unfilled ghost cells (level not covering)")
                for t in zip(*np.nonzero(need)):
                    c = tuple(gb[0][d] + t[d] for d in range(NDIM))
                    w = lvl.wrap(c)
                    cc = tuple(w[d] // rr[d] for d in range(NDIM))
                    cq = coarse.find(cc)
                    if cq < 0:
                        raise ValueError(f"ghost cell {c}: coarse parent {cc} not on the coarser level")
                    if cq not in refined:
                        refined[cq] = refine_patch_4d(data[l - 1][cq], rr, H.interp_mode)
                    fb0 = boxes.refine(coarse.boxes[cq], rr)[0]
                    fg[t] = refined[cq][tuple(w[d] - fb0[d] for d in range(NDIM))]
            # (iii) characteristic velocity boundary condition, v_x then v_y
            for vd in (2, 3):
                _apply_velocity_bc(fg, b, lvl, vd, E_bc[l], H.fbg[l])


def _vmask(shape, gb, lvl):
    """Cells of the ghosted box with both velocity indices inside the domain."""
    m = np.ones(shape, dtype=bool)
    for vd in (2, 3):
        idx = np.arange(gb[0][vd], gb[1][vd] + 1)
        ok = (idx >= lvl.domain[0][vd]) & (idx <= lvl.domain[1][vd])
        sh = [1] * NDIM
        sh[vd] = -1
        m &= ok.reshape(sh)
    return m


# --------------------------------------------------------------------------- reductions
def subpatch_moment(H, data):
    """Alg.8 (4D -> 2D): n = sum_l dvx_l dvy_l sum_v f on the finest (x, y) mesh (reading #13).
    x and y ghost cells of every level must be filled."""
    NX, NY = H.ncfg_finest()
    Rf = H.levels[-1].ratio
    total = np.zeros((NX, NY))
    partials = []
    for l, lvl in enumerate(H.levels):
        Rx, Ry = Rf[0] // lvl.ratio[0], Rf[1] // lvl.ratio[1]
        hl = H.h(l)
        dvv = hl[2] * hl[3]
        for p, b in enumerate(lvl.boxes):
            fg = data[l][p]
            nx, ny = boxes.size(b)[:2]
            pp = np.zeros((nx * Rx, ny * Ry))                # partial patch P_p
            for s in boxes.compute_sub_patches(b, l, H.levels):
                x0, x1 = s[0][0] - b[0][0], s[1][0] - b[0][0]
                y0, y1 = s[0][1] - b[0][1], s[1][1] - b[0][1]
                j0, j1 = s[0][2] - b[0][2], s[1][2] - b[0][2]
                m0, m1 = s[0][3] - b[0][3], s[1][3] - b[0][3]
                # grow by G in x and y, sum over the sub-patch's velocity range
                blk = fg[x0: x1 + 2 * G + 1, y0: y1 + 2 * G + 1, G + j0: G + j1 + 1, G + m0: G + m1 + 1]
                tmp = np.sum(blk, axis=(2, 3))
                fine = _refine_2d_interior(tmp, Rx, Ry)      # refine the 2D partial sums
                pp[x0 * Rx: (x1 + 1) * Rx, y0 * Ry: (y1 + 1) * Ry] += dvv * fine
            partials.append(((b[0][0] * Rx, b[0][1] * Ry), pp))
    for (x0, y0), pp in partials:                             # partial -> total (accumulate)
        total[x0: x0 + pp.shape[0], y0: y0 + pp.shape[1]] += pp
    return total


def covered_mask(H, l, p):
    """mu^p: 1 on cells of patch p not covered by level l+1 (4D), else 0."""
    b = H.levels[l].boxes[p]
    mu = np.ones(boxes.size(b))
    if l + 1 < len(H.levels):
        fl = H.levels[l + 1]
        rr = tuple(f // c for f, c in zip(fl.ratio, H.levels[l].ratio))
        for fb in fl.boxes:
            cb = boxes.intersect(boxes.coarsen(fb, rr), b)
            if not boxes.is_empty(cb):
                mu[_sl(cb, b[0])] = 0.0
    return mu


def mask_moment(H, data):
    """Alg.6 (4D -> 2D): every patch refined in x and y (linear5; interior velocity cells),
    covered cells masked, summed over both velocity dims into its partial patch, accumulated."""
    NX, NY = H.ncfg_finest()
    Rf = H.levels[-1].ratio
    total = np.zeros((NX, NY))
    partials = []
    for l, lvl in enumerate(H.levels):
        Rx, Ry = Rf[0] // lvl.ratio[0], Rf[1] // lvl.ratio[1]
        hl = H.h(l)
        dvv = hl[2] * hl[3]
        for p, b in enumerate(lvl.boxes):
            fg = data[l][p]
            nx, ny, nvx, nvy = boxes.size(b)
            blk = fg[:, :, G:G + nvx, G:G + nvy]             # ghosted x, y; interior v
            # refine in x then y (non-reduction dirs), one velocity cell at a time
            fine = np.empty((nx * Rx, ny * Ry, nvx, nvy))
            for j in range(nvx):
                for m in range(nvy):
                    fine[:, :, j, m] = _refine_2d_interior(blk[:, :, j, m], Rx, Ry)
            mu = np.repeat(np.repeat(covered_mask(H, l, p), Rx, axis=0), Ry, axis=1)
            pp = dvv * np.sum(mu * fine, axis=(2, 3))
            partials.append(((b[0][0] * Rx, b[0][1] * Ry), pp))
    for (x0, y0), pp in partials:
        total[x0: x0 + pp.shape[0], y0: y0 + pp.shape[1]] += pp
    return total


def inject(E_finest, R):
    """(2, NX, NY) finest field -> a level coarser by R = (R_x, R_y): mean of the R_x R_y finest
    cells."""
    c, NX, NY = E_finest.shape
    return np.asarray(E_finest).reshape(c, NX // R[0], R[0], NY // R[1], R[1]).mean(axis=(2, 4))


def constraints(H, data, reduction="subpatch"):
    """Reduction -> rho on the finest (x, y) mesh -> 2D Poisson -> E -> injection per level."""
    n = subpatch_moment(H, data) if reduction == "subpatch" else mask_moment(H, data)
    rho = 1.0 - n
    Rf = H.levels[-1].ratio
    E_f = field2d.efield_from_rho_2d(rho, H.h0[0] / Rf[0], H.h0[1] / Rf[1])
    return [inject(E_f, (Rf[0] // lvl.ratio[0], Rf[1] // lvl.ratio[1])) for lvl in H.levels], rho


# --------------------------------------------------------------------------- RHS / update
def patch_rhs(H, l, p, fg, E_l):
    b = H.levels[l].boxes[p]
    hl = H.h(l)
    n = boxes.size(b)
    vb = [scheme.exact_vbar(H.lower[2] + b[0][2] * hl[2], hl[2], n[2]),
          scheme.exact_vbar(H.lower[3] + b[0][3] * hl[3], hl[3], n[3])]
    Ep = []
    for c in range(2):
        Eg = field.ghost_periodic(E_l[c])
        Ep.append(Eg[b[0][0]: b[1][0] + 2 * G + 1, b[0][1]: b[1][1] + 2 * G + 1])
    return scheme.rhs(fg, vb, Ep, hl, H.recon)


def coarsen_fluxes_into(H, l, F_fine_lvl, F_coarse_lvl):
    """Alg.4: every coarse face that coincides with a face of a level-l patch takes the mean of
    the overlying fine F* over the transverse ratios (reading #14); periodic images in x, y."""
    fine, coarse = H.levels[l], H.levels[l - 1]
    rr = tuple(f // c for f, c in zip(fine.ratio, coarse.ratio))
    for q, fb in enumerate(fine.boxes):
        cfb = boxes.coarsen(fb, rr)
        for d in range(NDIM):
            Ff = F_fine_lvl[q][d]                          # faces along d: n_d + 1
            nf = boxes.size(fb)
            # fine faces that are coarse faces: local face index a with (fb.lo_d + a) % r_d == 0
            a_idx = [a for a in range(nf[d] + 1) if (fb[0][d] + a) % rr[d] == 0]
            for a in a_idx:
                sl = [slice(None)] * NDIM
                sl[d] = slice(a, a + 1)
                Fa = Ff[tuple(sl)]                         # (.., 1, ..) transverse fine faces
                shp = []
                for e in range(NDIM):
                    if e == d:
                        shp += [1]
                    else:
                        shp += [nf[e] // rr[e], rr[e]]
                mean = Fa.reshape(shp).mean(axis=tuple(2 * e + 1 - (1 if e > d else 0) for e in range(NDIM) if e != d))
                cface = (fb[0][d] + a) // rr[d]            # coarse face = low face of coarse cell cface
                for p, cb in enumerate(coarse.boxes):
                    Fc = F_coarse_lvl[p][d]
                    for s in (_images(coarse) if d < 2 else [(0, 0, 0, 0)]):
                        lo = [cfb[0][e] + s[e] for e in range(NDIM)]
                        hi = [cfb[1][e] + s[e] for e in range(NDIM)]
                        lo[d] = hi[d] = cface + s[d]
                        # coarse face index along d within patch cb: cface - cb.lo_d (0 .. n_d)
                        reg = []
                        ok = True
                        for e in range(NDIM):
                            lim_hi = cb[1][e] + 1 if e == d else cb[1][e]
                            a0, a1 = max(lo[e], cb[0][e]), min(hi[e], lim_hi)
                            if a0 > a1:
                                ok = False
                                break
                            reg.append((a0, a1))
                        if not ok:
                            continue
                        dst = tuple(slice(reg[e][0] - cb[0][e], reg[e][1] - cb[0][e] + 1) for e in range(NDIM))
                        src = tuple(slice(0, 1) if e == d else
                                    slice(reg[e][0] - lo[e], reg[e][1] - lo[e] + 1) for e in range(NDIM))
                        Fc[dst] = mean[src]


def average_down(H, data):
    """Coarse cells under a finer patch := mean of the fine cell averages, finest ->
    coarsest, in place on the interiors."""
    for l in range(len(H.levels) - 1, 0, -1):
        fine, coarse = H.levels[l], H.levels[l - 1]
        rr = tuple(f // c for f, c in zip(fine.ratio, coarse.ratio))
        for q, fb in enumerate(fine.boxes):
            ff = _interior(data[l][q])
            cbox = boxes.coarsen(fb, rr)
            n = boxes.size(cbox)
            mean = ff.reshape(n[0], rr[0], n[1], rr[1], n[2], rr[2], n[3], rr[3]).mean(axis=(1, 3, 5, 7))
            for p, cb in enumerate(coarse.boxes):
                ov = boxes.intersect(cb, cbox)
                if boxes.is_empty(ov):
                    continue
                _interior(data[l - 1][p])[_sl(ov, cb[0])] = mean[_sl(ov, cbox[0])]


def end_of_step_constraints(H, data, E_bc):
    fill_ghosts(H, data, E_bc)
    E_new, _ = constraints(H, data)
    return E_new


def step(H, data, E_bc, dt):
    """One synchronous RK4 step (Alg.5 with one hierarchy, Alg.1-4), as amr.step in 4D.
    Returns (new data, E(f_new), F*)."""
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
        E_lv, _ = constraints(H, pred)                                     # Alg.5
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


def start(H, data):
    """Ghosts with E_bc = 0, then the first constraint evaluation (Alg.5 start)."""
    zero = [np.zeros((2,) + tuple(H.ncells0[d] * lvl.ratio[d] for d in range(2))) for lvl in H.levels]
    fill_ghosts(H, data, zero)
    E, _ = constraints(H, data)
    return E
