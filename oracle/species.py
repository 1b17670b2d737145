"""Oracle: several species, one phase-space hierarchy each.  TEST INFRASTRUCTURE ONLY.

"Each species is represented by its own hierarchy ... the species are coupled only through the
configuration-space fields"; Alg.5 advances all hierarchies synchronously, evaluating
the constraints from all of them at every predictor state.  With species s of charge
q_s and mass m_s the system is (generalising P:191-217 with reading #1)

    f_s,t + v f_s,x + (q_s/m_s) E f_s,v = 0,   -phi_xx = rho = rho_bg + sum_s q_s int f_s dv,
    E = -phi_x.

The single-hierarchy oracle (amr.py) is the case of one species with q = -1, m = 1, rho_bg = 1
(electrons over immobile neutralising ions).  Here, for species s, the field entering its
phase-space update is A_s = -(q_s/m_s) E (so the electron case is A = E, as in scheme.rhs and the
v-boundary condition with a = -A), and the charge density sums the species' moments (Alg.8 per
hierarchy, on the common finest configuration mesh).
"""
from __future__ import annotations

import numpy as np

from . import amr, field, reduction, scheme

G = 2


class Species:
    def __init__(self, H, q, m):
        self.H = H
        self.q = float(q)
        self.m = float(m)


def charge_density(species, datas, rho_bg):
    """rho on the finest configuration mesh: rho_bg + sum_s q_s n_s, n_s the Alg.8 moment."""
    rho = None
    for sp, data in zip(species, datas):
        n = reduction.subpatch_moment(sp.H.levels, data, sp.H.h0[1], sp.H.ncells0[0])
        rho = (rho_bg + sp.q * n) if rho is None else rho + sp.q * n
    return rho


def constraints(species, datas, rho_bg):
    """Per species, per level: A_s = -(q_s/m_s) E injected; and rho."""
    H0 = species[0].H
    rho = charge_density(species, datas, rho_bg)
    dxf = H0.h0[0] / H0.levels[-1].ratio[0]
    E_f = field.efield_from_rho(rho, dxf)
    out = []
    for sp in species:
        rxf = sp.H.levels[-1].ratio[0]
        out.append([-(sp.q / sp.m) * reduction.inject(E_f, rxf // lvl.ratio[0]) for lvl in sp.H.levels])
    return out, rho


def start(species, datas, rho_bg):
    for sp, data in zip(species, datas):
        amr.fill_ghosts(sp.H, data, [np.zeros(sp.H.ncells0[0] * l.ratio[0]) for l in sp.H.levels])
    A, _ = constraints(species, datas, rho_bg)
    return A


def step(species, datas, A_bc, dt, rho_bg):
    """One synchronous RK4 step of all species (Alg.5 with several hierarchies, Alg.1-4 per
    hierarchy).  A_bc[s]: per-level effective field of species s from the previous constraint
    evaluation (reading #6b).  Returns (new datas, A_bc for the next step = the end-of-step
    constraint evaluation of Alg.5: ghosts of f_new with the stage-4 field, then
    the joint constraints)."""
    RK_ALPHA, RK_B = amr.RK_ALPHA, amr.RK_B
    f_old = [[[amr._interior(a).copy() for a in lvl] for lvl in data] for data in datas]
    k = [[[np.zeros_like(a) for a in lvl] for lvl in fo] for fo in f_old]
    F_acc = [[[None] * len(lvl.boxes) for lvl in sp.H.levels] for sp in species]
    for s in range(4):
        preds = []
        for i, sp in enumerate(species):                                   # Alg.2 per hierarchy
            pred = sp.H.new_data()
            for l in range(len(sp.H.levels)):
                for p in range(len(sp.H.levels[l].boxes)):
                    amr._interior(pred[l][p])[...] = f_old[i][l][p] + RK_ALPHA[s] * dt * k[i][l][p]
            amr.fill_ghosts(sp.H, pred, A_bc[i])
            preds.append(pred)
        A_lv, _ = constraints(species, preds, rho_bg)                      # Alg.5: all species
        for i, sp in enumerate(species):                                   # Alg.3 per hierarchy
            for l in range(len(sp.H.levels)):
                for p in range(len(sp.H.levels[l].boxes)):
                    k[i][l][p], F = amr.patch_rhs(sp.H, l, p, preds[i][l][p], A_lv[i][l])
                    F_acc[i][l][p] = [RK_B[s] * Fd for Fd in F] if F_acc[i][l][p] is None else \
                        [Fa + RK_B[s] * Fd for Fa, Fd in zip(F_acc[i][l][p], F)]
        A_bc = A_lv
    news = []
    for i, sp in enumerate(species):                                       # Alg.4 per hierarchy
        H = sp.H
        new = H.new_data()
        for l in range(len(H.levels) - 1, -1, -1):
            if l + 1 < len(H.levels):
                amr.coarsen_fluxes_into(H, l + 1, F_acc[i][l + 1], F_acc[i][l])
            for p in range(len(H.levels[l].boxes)):
                amr._interior(new[l][p])[...] = f_old[i][l][p] + dt * scheme.divergence(F_acc[i][l][p], H.h(l))
        amr.average_down(H, new)
        news.append(new)
    for i, sp in enumerate(species):                                       # Alg.5: constraints(f_new)
        amr.fill_ghosts(sp.H, news[i], A_bc[i])
    A_new, _ = constraints(species, news, rho_bg)
    return news, A_new
