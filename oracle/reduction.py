"""Oracle: velocity-moment reduction across a phase-space hierarchy (1D+1V).
TEST INFRASTRUCTURE ONLY.

rho_{i_c} = 1 - sum_l sum_p sum_j  dv_l  mu^p_i  I_x^{l,L-1} f^l_i

* reading #13: each level is weighted by its own dv_l (the printed V_v is outside the level sum),
* ``mask_reduce``     Alg.6 Mask Reduction: refine in x (linear5), mask
                      covered cells, sum over v into the partial patch; accumulate partial ->
                      total level,
* ``subpatch_reduce`` Alg.8 Sub-Patch Reduction: sub-patches by Alg.7, grow 2 cells
                      in x (reading #16), sum over v including those ghost columns, refine the 1D
                      partial sums in x, add into the partial patch (sub-patches of one patch may
                      share x-columns, e.g. below and above a finer patch, so their partial sums
                      are added -- "copy" of P:1255 read as accumulate), accumulate partial ->
                      total.

Hierarchy input: ``levels`` (list of boxes.LevelMeta, 1D+1V) and ``data[l][p]`` ghosted patch
arrays (G = 2) whose x-ghosts (rows) are filled.  ``dv0`` is the level-0 v spacing.
"""
from __future__ import annotations

import numpy as np

from . import boxes, interp

G = 2


def _finest_rx(levels):
    return levels[-1].ratio[0]


def covered_mask(levels, l, p):
    """mu^p: 1 on cells of patch p not covered by level l+1, else 0."""
    b = levels[l].boxes[p]
    nx, nv = boxes.size(b)
    mu = np.ones((nx, nv))
    if l + 1 < len(levels):
        fl = levels[l + 1]
        rr = tuple(f // c for f, c in zip(fl.ratio, levels[l].ratio))
        for fb in fl.boxes:
            cb = boxes.intersect(boxes.coarsen(fb, rr), b)
            if boxes.is_empty(cb):
                continue
            mu[cb[0][0] - b[0][0]: cb[1][0] - b[0][0] + 1,
               cb[0][1] - b[0][1]: cb[1][1] - b[0][1] + 1] = 0.0
    return mu


def _refine_x_rows(fg_rows, R):
    """linear5 refinement along x of ghosted rows: fg_rows (nx+2G, m) -> (nx*R, m)."""
    nx = fg_rows.shape[0] - 2 * G
    u5 = np.stack([fg_rows[a: a + nx] for a in range(5)], axis=-1)       # (nx, m, 5)
    fine = interp.linear5_1d(u5, R)                                      # (nx, m, R)
    return np.transpose(fine, (0, 2, 1)).reshape(nx * R, -1)


def mask_reduce(levels, data, dv0, nx0):
    """Alg.6.  Returns rho on the finest configuration mesh (length nx0 * finest ratio)."""
    rxf = _finest_rx(levels)
    total = np.zeros(nx0 * rxf)
    partials = []
    for l, lvl in enumerate(levels):
        R = rxf // lvl.ratio[0]
        dv = dv0 / lvl.ratio[1]
        for p, b in enumerate(lvl.boxes):
            nx, nv = boxes.size(b)
            fg = data[l][p]
            rows = fg[:, G:G + nv]                                # interior v, ghosted x
            fine = _refine_x_rows(rows, R)                        # refine in non-reduction dir
            mu = np.repeat(covered_mask(levels, l, p), R, axis=0)  # mask (constant per coarse cell)
            pp = dv * np.sum(mu * fine, axis=1)                   # sum reduce to partial patch
            partials.append((b[0][0] * R, pp))
    for x0, pp in partials:                                       # partial -> total (accumulate)
        total[x0: x0 + pp.size] += pp
    return 1.0 - total


def subpatch_reduce(levels, data, dv0, nx0):
    """Alg.8.  Returns rho = 1 - n on the finest configuration mesh (electrons over the immobile
    neutralising background)."""
    return 1.0 - subpatch_moment(levels, data, dv0, nx0)


def subpatch_moment(levels, data, dv0, nx0, first=False, vlo=0.0):
    """Alg.8 velocity moment n = sum_l dv_l sum_v f (reading #13) on the finest configuration mesh.
    first=True: the first moment sum_l dv_l sum_v <v f> instead (N4 current, reading #31): per
    sub-patch column the fourth-order product rule sum_j vbar_j f_j + (dv/24)(f_{j1+1} + f_{j1} -
    f_{j0} - f_{j0-1}) over its velocity range j0..j1 (the telescoped (dv/24)(f_{j+1} - f_{j-1})),
    vbar_j the exact cell-average velocity of level cell j, vlo the domain's lower velocity."""
    rxf = _finest_rx(levels)
    total = np.zeros(nx0 * rxf)
    partials = []
    for l, lvl in enumerate(levels):
        R = rxf // lvl.ratio[0]
        dv = dv0 / lvl.ratio[1]
        for p, b in enumerate(lvl.boxes):
            nx, nv = boxes.size(b)
            fg = data[l][p]
            pp = np.zeros(nx * R)                                 # partial patch P_p
            for s in boxes.compute_sub_patches(b, l, levels):
                x0, x1 = s[0][0] - b[0][0], s[1][0] - b[0][0]     # patch-local interior x range
                j0, j1 = s[0][1] - b[0][1], s[1][1] - b[0][1]
                # grow by G in x, sum over the sub-patch v range including the ghost columns
                rows = fg[G + x0 - G: G + x1 + G + 1, :]
                if first:
                    vbar = vlo + (b[0][1] + np.arange(j0, j1 + 1) + 0.5) * dv
                    tmp = rows[:, G + j0: G + j1 + 1] @ vbar + (dv / 24.0) * (
                        rows[:, G + j1 + 1] + rows[:, G + j1] - rows[:, G + j0] - rows[:, G + j0 - 1])
                else:
                    tmp = np.sum(rows[:, G + j0: G + j1 + 1], axis=1)
                fine = _refine_x_rows(tmp[:, None], R)[:, 0]      # refine the 1D partial sums
                pp[x0 * R: (x1 + 1) * R] += dv * fine             # into the partial patch
            partials.append((b[0][0] * R, pp))
    for x0, pp in partials:
        total[x0: x0 + pp.size] += pp
    return total


def inject(E_finest, rx_finest_over_level):
    """Injection of the finest configuration field into a level whose x
    resolution is coarser by R: mean of the R finest values (config mesh uniform at the finest
    x resolution and averaged down to coarser levels).  No ghosts."""
    R = rx_finest_over_level
    return np.mean(np.asarray(E_finest).reshape(-1, R), axis=1)
