"""Oracle-side drivers of the multi-level runs used by the AMR parity tests (test infrastructure:
imports oracle/ and inputs/ only).  They follow the same protocol as
paper_1204_3853_b200.amr_solver.AmrVlasov1D:

* start: interiors set, ghosts filled with E_bc = 0, E_bc := constraints(f) (Alg.5 start);
* regrid (C3 rule, reading #18): ghosts filled with E_bc, tags on level 0, dilation, fixed tiles,
  new fine data copied from the old fine level where it overlaps, else interpolated from level 0;
  then ghosts filled with E_bc (kept for surviving levels, zero for a new level) and
  E_bc := constraints(new hierarchy) (Alg.5 evaluates the constraints after regridHierarchies).
"""
from __future__ import annotations

import numpy as np

import inputs
from oracle import amr, boxes, interp, scheme


def hierarchy(w, level_boxes, ratios, recon=scheme.CENTERED4, mode=interp.LINEAR5):
    return amr.Hierarchy(w.lower, inputs.spacing(w), w.ncells,
                         [[boxes.box(*b) for b in bl] for bl in level_boxes], ratios,
                         lambda r: inputs.background_profile(w, r), recon, mode)


def zero_E(H):
    return [np.zeros(H.ncells0[0] * lvl.ratio[0]) for lvl in H.levels]


def start(H, data):
    amr.fill_ghosts(H, data, zero_E(H))
    E_bc, _ = amr.constraints(H, data)
    return E_bc


def regrid(H, data, E_bc, tol, buffer, ratio, tile, clustered=None):
    """clustered: None (C3 fixed tiles) or (smallest, largest, efficiency) in level-1 cells."""
    amr.fill_ghosts(H, data, E_bc)
    nlev_old = len(H.levels)
    tags = amr.level0_tags(H, data, tol)
    if clustered is None:
        new, new_boxes = amr.regrid_two_level(H, data, E_bc, tol, buffer, ratio, tile)
    else:
        new, new_boxes = amr.regrid_two_level_clustered(H, data, E_bc, tol, buffer, ratio, *clustered)
    E_fill = [E_bc[0]]
    if new_boxes:
        E_fill.append(E_bc[1] if nlev_old > 1 else np.zeros(H.ncells0[0] * ratio[0]))
    amr.fill_ghosts(H, new, E_fill)
    E_new, _ = amr.constraints(H, new)
    return new, E_new, new_boxes, tags


def next_dt(H, E_bc, dt_prev, cfl=0.5, growth=1.1):
    """Adaptive step (reading #17): min(cfl / max_l(max|vbar|/dx_l + max|E_l|/dv_l),
    growth * dt_prev), vbar over the finest level's whole velocity range."""
    hf = H.h(len(H.levels) - 1)
    nv = H.ncells0[1] * H.levels[-1].ratio[1]
    vmax = max(abs(H.lower[1] + 0.5 * hf[1]), abs(H.lower[1] + (nv - 0.5) * hf[1]))
    rate = max(vmax / H.h(l)[0] + np.max(np.abs(E_bc[l])) / H.h(l)[1] for l in range(len(H.levels)))
    return min(cfl / rate, growth * dt_prev)


def c3_run(w, nsteps, regrid_every, dt, tol, buffer, ratio, tile, recon=scheme.CENTERED4, mode=interp.LINEAR5,
           log=None, clustered=None, adaptive=False):
    """Two-level run from level 0 only: regrid at step 0 and every `regrid_every` steps."""
    lb0 = inputs.level0_boxes(w)
    H = hierarchy(w, [lb0], [(1, 1)], recon, mode)
    data = H.new_data()
    for p, b in enumerate(H.levels[0].boxes):
        data[0][p][2:-2, 2:-2] = inputs.initial_cell_averages(w, (1, 1), b)
    E_bc = start(H, data)
    for n in range(nsteps):
        if n % regrid_every == 0:
            data, E_bc, nb, tags = regrid(H, data, E_bc, tol, buffer, ratio, tile, clustered)
            if log is not None:
                log.append((n, [tuple(map(tuple, b)) for b in nb], tags))
        data, E_bc, _ = amr.step(H, data, E_bc, dt)
        if adaptive:
            dt = next_dt(H, E_bc, dt)
            if log is not None:
                log.append(("dt", dt))
    return H, data, E_bc


def regrid_multilevel(H, data, E_bc, tol, buffers, ratios, smallest, largest, efficiency=0.7):
    """Oracle side of AmrVlasov1D.regrid_hierarchy: multi-level regrid, then ghosts (E_bc kept for
    surviving level indices with the same ratio, 0 for new ones) and the constraints."""
    old_ratios = [l.ratio for l in H.levels]
    new, nbs = amr.regrid_hierarchy(H, data, E_bc, tol, buffers, ratios, smallest, largest, efficiency)
    E_fill = [E_bc[l] if (l < len(E_bc) and l < len(old_ratios) and old_ratios[l] == H.levels[l].ratio)
              else np.zeros(H.ncells0[0] * H.levels[l].ratio[0]) for l in range(len(H.levels))]
    amr.fill_ghosts(H, new, E_fill)
    E_new, _ = amr.constraints(H, new)
    return new, E_new, nbs
