"""Oracle: fourth-order finite-volume phase-space right-hand side.  TEST INFRASTRUCTURE ONLY.

Follows PAPER.md section 2 literally:

  d f_ij/dt = -(<vf>_{i+1/2,j} - <vf>_{i-1/2,j})/dx + (<Ef>_{i,j+1/2} - <Ef>_{i,j-1/2})/dv

  <vf>_{i+1/2,j} = vbar_j <f>_{i+1/2,j} + (dv/24)(<f>_{i+1/2,j+1} - <f>_{i+1/2,j-1})
  <Ef>_{i,j+1/2} = Ebar_i <f>_{i,j+1/2} + (1/48)(Ebar_{i+1}-Ebar_{i-1})(<f>_{i+1,j+1/2}-<f>_{i-1,j+1/2})
                   (printed "-1/48": reading #3 takes +1/48)

  <f>_{i+1/2} = w_L (-f_{i-1} + 5 f_i + 2 f_{i+1})/6 + w_R (2 f_i + 5 f_{i+1} - f_{i+2})/6
  CENTERED4: w_L = w_R = 1/2.  UPWIND: provisional WENO weights (reading #4), the
  larger one given to the upwind stencil.

Generalised dimension by dimension to 2D+2V (BASELINE.json C5): a configuration-space face
along x_d carries one transverse term along v_d (v_d is the only coordinate its coefficient
depends on); a velocity-space face along v_d carries one (1/48) product term per configuration
dim (E_d depends on all of x).  This is the same product rule <ab> = a b + (h^2/12) grad a . grad b
that gives P:265-273 in 1D+1V.

Array conventions: phase-space arrays are *ghosted* (G = 2 cells on every side), axes ordered
configuration dims first then velocity dims.
"""
from __future__ import annotations

import numpy as np

G = 2
CENTERED4 = "centered4"
UPWIND = "upwind"
EPS_WENO = 1.0e-6   # P:762 "typically epsilon = 10^-6" (reading #4 borrows it for face weights)


# --------------------------------------------------------------------------- faces
def third_order_left(fm1, f0, fp1):
    """Eq. (thirdLeft)."""
    return (-fm1 + 5.0 * f0 + 2.0 * fp1) / 6.0


def third_order_right(f0, fp1, fp2):
    """Eq. (thirdRight)."""
    return (2.0 * f0 + 5.0 * fp1 - fp2) / 6.0


def provisional_weights(fm1, f0, fp1, fp2):
    """Provisional weights hat w_L, hat w_R by "the standard WENO methodology".
    Reading #4 (mirror-symmetric smoothness indicators of the two 3-cell stencils, ideal
    weights 1/2, eps = 1e-6)."""
    beta_l = (13.0 / 12.0) * (fm1 - 2.0 * f0 + fp1) ** 2 + 0.25 * (fp1 - fm1) ** 2
    beta_r = (13.0 / 12.0) * (f0 - 2.0 * fp1 + fp2) ** 2 + 0.25 * (fp2 - f0) ** 2
    alpha_l = 0.5 / (EPS_WENO + beta_l) ** 2
    alpha_r = 0.5 / (EPS_WENO + beta_r) ** 2
    return alpha_l / (alpha_l + alpha_r), alpha_r / (alpha_l + alpha_r)


def face_average(fm1, f0, fp1, fp2, recon, upwind):
    """<f> on the face between cells (f0, fp1), eq. (limitedFace) P:329.

    ``upwind`` is the advection velocity on the face (v_j for x-faces, a_i = -E_i for v-faces);
    if it is > 0 the left (lower) stencil is upwind and receives max(hat w)."""
    left = third_order_left(fm1, f0, fp1)
    right = third_order_right(f0, fp1, fp2)
    if recon == CENTERED4:
        return 0.5 * left + 0.5 * right
    if recon != UPWIND:
        raise ValueError(recon)
    wl_hat, wr_hat = provisional_weights(fm1, f0, fp1, fp2)
    big = np.maximum(wl_hat, wr_hat)
    small = np.minimum(wl_hat, wr_hat)
    pos = np.asarray(upwind) > 0
    w_l = np.where(pos, big, small)
    w_r = np.where(pos, small, big)
    return w_l * left + w_r * right


# --------------------------------------------------------------------------- helpers
def _sl(ndim, axis, s):
    idx = [slice(None)] * ndim
    idx[axis] = s
    return tuple(idx)


def _bcast(vec, ndim, axes):
    """Reshape ``vec`` (with len(axes) dims) to broadcast over ``ndim`` dims on ``axes``."""
    shape = [1] * ndim
    for a, n in zip(axes, vec.shape):
        shape[a] = n
    return vec.reshape(shape)


def all_face_averages(fg, axis, recon, upwind):
    """Face averages along ``axis`` for every face whose 4-cell stencil lies in the ghosted
    array.  Entry m (along ``axis``) is the face between ghosted cells m+1 and m+2."""
    n = fg.shape[axis]
    c = [fg[_sl(fg.ndim, axis, slice(a, n - 3 + a))] for a in range(4)]
    return face_average(c[0], c[1], c[2], c[3], recon, upwind)


def _interior(fa, face_axis, n, shifts=None):
    """Slice of a face array: along ``face_axis`` the n+1 faces bounding interior cells
    (ghosted cells G..G+n-1 -> face entries G-2..G+n-2); other axes interior, shifted by
    ``shifts[axis]`` cells (for the transverse terms)."""
    shifts = shifts or {}
    idx = []
    for a in range(fa.ndim):
        if a == face_axis:
            idx.append(slice(G - 2, G + n[a] - 1))
        else:
            s = shifts.get(a, 0)
            idx.append(slice(G + s, G + n[a] + s))
    return fa[tuple(idx)]


# --------------------------------------------------------------------------- fluxes
def fluxes(fg, vbar, E, h, recon):
    """Face-averaged fluxes on all faces of the interior cells.

    fg    ghosted cell averages, shape (n_0+2G, ..., n_{D-1}+2G), D = 2*ncfg
    vbar  list (one per velocity dim) of ghosted exact cell-average velocities
    E     list (one per velocity dim) of ghosted cell-averaged field components, each of the
          ghosted configuration-space shape
    h     mesh spacings per dim
    Returns F[d] for every axis d: shape = interior shape with n_d + 1 faces along d.
    F[d] is <v_d f> for configuration axes and <E_d f> for velocity axes."""
    ndim = fg.ndim
    ncfg = ndim // 2
    n = [s - 2 * G for s in fg.shape]
    cfg_axes = list(range(ncfg))
    out = []
    for d in range(ndim):
        if d < ncfg:
            vd = ncfg + d
            upw = _bcast(vbar[d], ndim, [vd])
            fa = all_face_averages(fg, d, recon, upw)
            vb = _bcast(vbar[d][G:G + n[vd]], ndim, [vd])
            flux = vb * _interior(fa, d, n) + (h[vd] / 24.0) * (
                _interior(fa, d, n, {vd: +1}) - _interior(fa, d, n, {vd: -1}))
        else:
            e = E[d - ncfg]
            upw = _bcast(-e, ndim, cfg_axes)          # a = -E (reading #1 / #30)
            fa = all_face_averages(fg, d, recon, upw)
            e_int = e[tuple(slice(G, G + n[c]) for c in cfg_axes)]
            flux = _bcast(e_int, ndim, cfg_axes) * _interior(fa, d, n)
            for c in cfg_axes:
                ep = e[tuple(slice(G + (1 if a == c else 0), G + n[a] + (1 if a == c else 0)) for a in cfg_axes)]
                em = e[tuple(slice(G - (1 if a == c else 0), G + n[a] - (1 if a == c else 0)) for a in cfg_axes)]
                flux = flux + (1.0 / 48.0) * _bcast(ep - em, ndim, cfg_axes) * (
                    _interior(fa, d, n, {c: +1}) - _interior(fa, d, n, {c: -1}))
        out.append(flux)
    return out


def divergence(F, h):
    """Right-hand side of the semi-discrete system from face fluxes:
    -sum_cfg (F_hi - F_lo)/h + sum_vel (F_hi - F_lo)/h."""
    ndim = len(F)
    ncfg = ndim // 2
    k = None
    for d in range(ndim):
        hi = F[d][_sl(ndim, d, slice(1, None))]
        lo = F[d][_sl(ndim, d, slice(None, -1))]
        term = (hi - lo) / h[d]
        term = -term if d < ncfg else term
        k = term if k is None else k + term
    return k


def rhs(fg, vbar, E, h, recon):
    """k = L(f) and the fluxes it was built from (Alg.3 computeFluxes + fluxDivergence)."""
    F = fluxes(fg, vbar, E, h, recon)
    return divergence(F, h), F


def exact_vbar(lower, h, n):
    """Exact cell-average velocities on the ghosted range of n cells:
    vbar_j = (v_{j-1/2} + v_{j+1/2})/2 for j = -G..n-1+G."""
    j = np.arange(-G, n + G, dtype=np.float64)
    return 0.5 * ((lower + j * h) + (lower + (j + 1.0) * h))
