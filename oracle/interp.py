"""Oracle: conservative cell-average interpolation coarse -> fine.  TEST INFRASTRUCTURE ONLY.

linear5: fine averages u^f_{Ri+s} = sum_{j=-2..2} b_j(s) u_{i+j}, with b_j(s) the
  sub-cell averages of the quintic-stencil interpolant gamma_j(eta).  The printed b_j formulas
   are used as printed, with p_k(s) = [(s+1)^{k+1} - s^{k+1}] / R^k (reading #12: the
  printed p_k has no R and the wrong binomial sum; this p_k is (k+1) x the mean of
  eta^k over the sub-cell [s/R, (s+1)/R]).
WENO5: smoothness detectors beta^(r), weights alpha^(r), omega^(r), candidate
  sub-cell averages A + B (2s+1)/(2R) + C (3s^2+3s+1)/(6R^2), renormalised to the coarse mean.
  Readings: #8 B^(0) = 2D_i - D_{i+1} (printed 2D_i - D_{i-1}); #10 the conservation defect is
  added to every sub-cell (printed: last sub-cell only; prose: "equidistributed").
Multi-D: dimension by dimension, x (axis 0) first, then v.
"""
from __future__ import annotations

from fractions import Fraction

import numpy as np

EPS_WENO = 1.0e-6
D_IDEAL = (0.3, 0.6, 0.1)            # P:761 d_0 = 3/10, d_1 = 3/5, d_2 = 1/10
LINEAR5 = "linear5"
WENO5 = "weno5"


# --------------------------------------------------------------------------- linear5
def p_k(k, s, R):
    """p_k(s) (reading #12), as an exact Fraction."""
    s = Fraction(s)
    return ((s + 1) ** (k + 1) - s ** (k + 1)) / Fraction(R) ** k


def linear5_weights_exact(R):
    """b_j(s), j = -2..2, s = 0..R-1, exact rationals."""
    rows = []
    for s in range(R):
        p1, p2, p3, p4 = (p_k(k, s, R) for k in (1, 2, 3, 4))
        b_m2 = (p4 - 5 * p3 + 5 * p2 + 5 * p1 - 6) / 120
        b_m1 = (-4 * p4 + 15 * p3 + 10 * p2 - 75 * p1 + 54) / 120
        b_0 = (6 * p4 - 15 * p3 - 40 * p2 + 75 * p1 + 94) / 120
        b_p1 = (-4 * p4 + 5 * p3 + 30 * p2 - 5 * p1 - 26) / 120
        b_p2 = (p4 - 5 * p2 + 4) / 120
        rows.append((b_m2, b_m1, b_0, b_p1, b_p2))
    return rows


def linear5_weights(R):
    """b_j(s) as fp64, shape (R, 5)."""
    return np.array([[float(x) for x in row] for row in linear5_weights_exact(R)])


def linear5_1d(u5, R):
    """u5[..., 5] = u_{i-2..i+2} -> [..., R] fine averages."""
    b = linear5_weights(R)
    u5 = np.asarray(u5, dtype=np.float64)
    out = np.zeros(u5.shape[:-1] + (R,))
    for s in range(R):
        acc = np.zeros(u5.shape[:-1])
        for j in range(5):
            acc = acc + b[s, j] * u5[..., j]
        out[..., s] = acc
    return out


# --------------------------------------------------------------------------- WENO5
def weno5_1d(u5, R):
    """Limited conservative interpolation of P:741-831 for one coarse cell i given
    u5[..., 0..4] = u_{i-2..i+2}; returns [..., R] fine averages u^f_{Ri+s}."""
    u = np.asarray(u5, dtype=np.float64)
    um2, um1, u0, up1, up2 = (u[..., m] for m in range(5))
    # (aux1) D_{i+n}, n = -2..1 and Delta_{i+p}, p = -1..1
    D_m2 = um1 - um2
    D_m1 = u0 - um1
    D_0 = up1 - u0
    D_p1 = up2 - up1
    Dl_m1 = D_m1 - D_m2
    Dl_0 = D_0 - D_m1
    Dl_p1 = D_p1 - D_0
    # step 1: smoothness detectors
    beta = (
        (13.0 / 12.0) * Dl_p1 ** 2 + 0.25 * (D_p1 - 3.0 * D_0) ** 2,
        (13.0 / 12.0) * Dl_0 ** 2 + 0.25 * (D_0 + D_m1) ** 2,
        (13.0 / 12.0) * Dl_m1 ** 2 + 0.25 * (3.0 * D_m1 - D_m2) ** 2,
    )
    # steps 2-3: absolute and relative weights
    alpha = [D_IDEAL[r] / (EPS_WENO + beta[r]) ** 2 for r in range(3)]
    asum = alpha[0] + alpha[1] + alpha[2]
    omega = [alpha[r] / asum for r in range(3)]
    # (aux2)
    A = (u0 + (2.0 * D_p1 - 5.0 * D_0) / 6.0,
         u0 - (D_0 + 2.0 * D_m1) / 6.0,
         u0 - (4.0 * D_m1 - D_m2) / 6.0)
    B = (2.0 * D_0 - D_p1, D_m1, D_m1)                     # reading #8 for B^(0)
    C = (Dl_p1, Dl_0, Dl_m1)
    out = np.zeros(u.shape[:-1] + (R,))
    for s in range(R):
        bs = (2.0 * s + 1.0) / (2.0 * R)
        cs = (3.0 * s * s + 3.0 * s + 1.0) / (6.0 * R * R)
        val = np.zeros(u.shape[:-1])
        for r in range(3):
            val = val + omega[r] * (A[r] + B[r] * bs + C[r] * cs)   # eq. (interp_r_avg) + step 5
        out[..., s] = val
    # renormalisation to the coarse average (reading #10: defect added to every sub-cell)
    defect = u0 - np.mean(out, axis=-1)
    return out + defect[..., None]


def interp_1d(u5, R, mode):
    if mode == LINEAR5:
        return linear5_1d(u5, R)
    if mode == WENO5:
        return weno5_1d(u5, R)
    raise ValueError(mode)


def interp_fine_cell_2d(coarse5x5, Rx, Rv, sx, sv, mode):
    """Fine cell (sx, sv) of the coarse cell at the centre of the 5x5 coarse block
    coarse5x5[a, b] = u_{i-2+a, j-2+b}: first x (for each of the 5 coarse v-columns),
    then v on the partially refined values."""
    partial = np.array([interp_1d(coarse5x5[:, b], Rx, mode)[sx] for b in range(5)])
    return interp_1d(partial, Rv, mode)[sv]


def refine_patch_2d(coarse_ghosted, Rx, Rv, mode, g=2):
    """Refine every interior coarse cell of a ghosted (g >= 2) 2D array: returns the fine
    array (Rx*nx, Rv*nv).  Dimension by dimension: x pass on all coarse v-columns (interior
    and ghosts) then v pass."""
    cg = np.asarray(coarse_ghosted, dtype=np.float64)
    nx, nv = cg.shape[0] - 2 * g, cg.shape[1] - 2 * g
    # x pass: for coarse rows i, all ghosted columns
    u5 = np.stack([cg[g - 2 + a: g - 2 + a + nx, :] for a in range(5)], axis=-1)  # (nx, nvg, 5)
    xp = interp_1d(u5, Rx, mode)                                                  # (nx, nvg, Rx)
    xp = np.transpose(xp, (0, 2, 1)).reshape(nx * Rx, -1)                         # (nx*Rx, nvg)
    v5 = np.stack([xp[:, g - 2 + b: g - 2 + b + nv] for b in range(5)], axis=-1)  # (nx*Rx, nv, 5)
    fp = interp_1d(v5, Rv, mode)                                                  # (nx*Rx, nv, Rv)
    return fp.reshape(nx * Rx, nv * Rv)
