"""Oracle: velocity moment, periodic 1D Poisson solve and cell-averaged E.  TEST INFRASTRUCTURE ONLY.

  rho_i = 1 - dv * sum_j f_ij
  30 phi_i - 16 (phi_{i+1} + phi_{i-1}) + (phi_{i+2} + phi_{i-2}) = 12 dx^2 rho_i
        (printed "12 dx": reading #2 takes dx^2)
  periodic null space: project rho to mean zero; phi normalised to mean zero
  E_i = -[8 (phi_{i+1} - phi_{i-1}) - phi_{i+2} + phi_{i-2}] / (12 dx)
        (printed with "+": reading #1 takes E = -d_x phi, consistent with
         P:192)

The linear system is LU-factorised once per (n, dx) and stored.  The singular
periodic matrix is made regular by bordering it with the constraint sum(phi) = 0.
"""
from __future__ import annotations

import functools

import numpy as np
import scipy.linalg as sla

G = 2


def moment_rho(f_interior, dv_volume):
    """rho = 1 - V_v sum over all velocity cells (V_v = product of velocity spacings,
    P:1072).  Velocity axes are the trailing half of the axes."""
    ndim = f_interior.ndim
    vel_axes = tuple(range(ndim // 2, ndim))
    return 1.0 - dv_volume * np.sum(f_interior, axis=vel_axes)


def poisson_matrix(n):
    """Periodic pentadiagonal matrix of eq. (discrete_potential)."""
    if n < 5:
        raise ValueError("periodic 5-point Poisson needs n >= 5")
    A = np.zeros((n, n))
    for i in range(n):
        A[i, i] = 30.0
        A[i, (i + 1) % n] += -16.0
        A[i, (i - 1) % n] += -16.0
        A[i, (i + 2) % n] += 1.0
        A[i, (i - 2) % n] += 1.0
    return A


@functools.lru_cache(maxsize=16)
def _bordered_lu(n):
    """LU factors of [[A, 1], [1^T, 0]] (A periodic, singular with null space = constants)."""
    A = poisson_matrix(n)
    B = np.zeros((n + 1, n + 1))
    B[:n, :n] = A
    B[:n, n] = 1.0
    B[n, :n] = 1.0
    return sla.lu_factor(B)


def solve_potential(rho, dx):
    """Mean-zero phi solving the periodic system with the projected rho."""
    rho = np.asarray(rho, dtype=np.float64)
    n = rho.size
    rho_proj = rho - rho.mean()                       # project out the null-space component
    rhs = np.concatenate([12.0 * dx * dx * rho_proj, [0.0]])
    sol = sla.lu_solve(_bordered_lu(n), rhs)
    return sol[:n]


def efield_from_potential(phi, dx):
    """E_i = -D4 phi (reading #1), periodic."""
    p = lambda s: np.roll(phi, -s)   # p(s)[i] = phi[i+s]
    return -(8.0 * (p(1) - p(-1)) - p(2) + p(-2)) / (12.0 * dx)


def efield_from_rho(rho, dx):
    return efield_from_potential(solve_potential(rho, dx), dx)


def ghost_periodic(a, g=G):
    """Periodic ghost extension of a configuration-space array along every axis."""
    return np.pad(a, [(g, g)] * a.ndim, mode="wrap")


def current_density(f_ghosted, v_lo, dv, q=-1.0, g=G):
    """Current moment j_i = q dv sum_j <v f>_ij of one species on a uniform 1D+1V level (N4, toward
    Vlasov-Maxwell; reading #31): the fourth-order cell average of the product v f by the
    same product rule as the fluxes (reading #3),
        <v f>_j = vbar_j fbar_j + (dv / 24) (fbar_{j+1} - fbar_{j-1}),   vbar_j = v_lo + (j + 1/2) dv,
    with fbar_{-1}, fbar_{nv} the velocity ghost values.  f_ghosted: (nx + 2g, nv + 2g)."""
    f = np.asarray(f_ghosted, dtype=np.float64)[g:-g, :]
    nv = f.shape[1] - 2 * g
    vbar = v_lo + (np.arange(nv) + 0.5) * dv
    vf = vbar[None, :] * f[:, g:g + nv] + (dv / 24.0) * (f[:, g + 1:g + 1 + nv] - f[:, g - 1:g - 1 + nv])
    return q * dv * vf.sum(axis=1)
