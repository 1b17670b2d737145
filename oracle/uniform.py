"""Oracle: single-level (uniform) Vlasov advance.  TEST INFRASTRUCTURE ONLY.

* Domain and boundary conditions: configuration dims periodic; velocity dims
  truncated with a characteristic condition -- outgoing characteristics extrapolated, incoming
  ones carry the unperturbed profile.  Reading #6: outgoing => cubic extrapolation of the cell
  averages (exact for cubic data), incoming or zero => exact cell averages of the unperturbed
  profile (passed in as ``fbg``).  The characteristic speed along v_d is a_d = -E_d.
* Time advance: classic RK4 in the flux-accumulation form, organised
  as Alg.1-5 for one hierarchy with one level:
      for s = 1..4:  f_pred = f_old + alpha_s dt k        (ComputePredictorState, Alg.2)
                     fill ghosts + BC with E_bc            (Alg.2)
                     E = constraints(f_pred); E_bc = E     (Alg.5)
                     k, F = RHS(f_pred, E); F* += b_s F    (Alg.3)
      f_new = f_old + dt * div(F*)                         (Alg.4)
  Reading #6b: Alg.5 evaluates the predictor state (with its boundary condition)
  BEFORE the constraints, so the boundary condition of a predictor state uses the E of the
  previous constraint evaluation: stage s >= 2 the E of stage s-1; stage 1 the E of the
  end-of-step ComputeInstantaneousConstraints(f_new) of the previous step, i.e. E(f_n) (at
  n = 0 the initial evaluation E(f_0)).  On one periodic level the moment does not read ghost
  cells, so E(f_n) is also the stage-1 field: stage 1 uses E_bc = E.
"""
from __future__ import annotations

import numpy as np

from . import field, scheme

G = 2
RK_ALPHA = (0.0, 0.5, 0.5, 1.0)
RK_B = (1.0 / 6.0, 1.0 / 3.0, 1.0 / 3.0, 1.0 / 6.0)
RK_C = (0.0, 0.5, 0.5, 1.0)


def _sl(ndim, axis, s):
    idx = [slice(None)] * ndim
    idx[axis] = s
    return tuple(idx)


def extrapolate_low(f0, f1, f2, f3):
    """Ghosts -1, -2 by cubic extrapolation of the first four cells (reading #6)."""
    return 4.0 * f0 - 6.0 * f1 + 4.0 * f2 - f3, 10.0 * f0 - 20.0 * f1 + 15.0 * f2 - 4.0 * f3


def apply_velocity_bc(fg, E_bc, fbg, vaxis):
    """Fill the 2 ghost layers of velocity axis ``vaxis`` in place (all other indices over
    their full ghosted range).  E_bc[d]: ghosted configuration arrays; fbg: unperturbed
    profile cell averages on the ghosted velocity range (1D for 1V, 2D for 2V)."""
    ndim = fg.ndim
    ncfg = ndim // 2
    comp = vaxis - ncfg
    n = fg.shape[vaxis] - 2 * G
    a = -E_bc[comp]                                              # characteristic speed
    a = a.reshape(a.shape + (1,) * (ndim - ncfg))                # broadcast over velocity axes
    cell = lambda j: fg[_sl(ndim, vaxis, slice(G + j, G + j + 1))]
    # profile values of the ghost layers, broadcast over configuration axes
    prof = fbg.reshape((1,) * ncfg + fbg.shape)
    pg = lambda j: prof[_sl(ndim, vaxis, slice(G + j, G + j + 1))]
    # low side: outgoing if a < 0
    g1, g2 = extrapolate_low(cell(0), cell(1), cell(2), cell(3))
    out = a < 0
    fg[_sl(ndim, vaxis, slice(G - 1, G))] = np.where(out, g1, pg(-1))
    fg[_sl(ndim, vaxis, slice(G - 2, G - 1))] = np.where(out, g2, pg(-2))
    # high side: outgoing if a > 0 (mirror image of the low-side formula)
    g1, g2 = extrapolate_low(cell(n - 1), cell(n - 2), cell(n - 3), cell(n - 4))
    out = a > 0
    fg[_sl(ndim, vaxis, slice(G + n, G + n + 1))] = np.where(out, g1, pg(n))
    fg[_sl(ndim, vaxis, slice(G + n + 1, G + n + 2))] = np.where(out, g2, pg(n + 1))


def fill_ghosts_uniform(f, E_bc, fbg):
    """Ghosted copy of a periodic single-patch level: configuration axes wrap periodically
    (exchange across the periodic boundary, Alg.2), then each velocity axis in order gets the
    characteristic boundary condition over the full ghosted extent of the other axes."""
    ndim = f.ndim
    ncfg = ndim // 2
    fg = np.full(tuple(s + 2 * G for s in f.shape), np.nan)
    inner = tuple(slice(G, G + s) for s in f.shape)
    fg[inner] = f
    # periodic configuration axes (interior velocity range)
    for c in range(ncfg):
        n = f.shape[c]
        sel = [slice(None)] * ndim
        for v in range(ncfg, ndim):
            sel[v] = slice(G, G + f.shape[v])
        lo_dst = list(sel); lo_dst[c] = slice(0, G)
        lo_src = list(sel); lo_src[c] = slice(n, n + G)
        hi_dst = list(sel); hi_dst[c] = slice(n + G, n + 2 * G)
        hi_src = list(sel); hi_src[c] = slice(G, 2 * G)
        fg[tuple(lo_dst)] = fg[tuple(lo_src)]
        fg[tuple(hi_dst)] = fg[tuple(hi_src)]
    for v in range(ncfg, ndim):
        apply_velocity_bc(fg, E_bc, fbg, v)
    return fg


class UniformProblem:
    """A periodic single-level problem: geometry + field mode.

    lower, h      physical lower corner and spacings per axis
    shape         interior cells per axis
    fbg           unperturbed velocity profile on the ghosted velocity range
    field_mode    'poisson' (E from the periodic Poisson solve: 1D, or 2D for 2D+2V, field2d) or
                  'prescribed'
    E_prescribed  (ncfg, *cfg_shape) cell-averaged field for 'prescribed'
    """

    def __init__(self, lower, h, shape, fbg, recon=scheme.CENTERED4, field_mode="poisson",
                 E_prescribed=None):
        self.lower = tuple(float(x) for x in lower)
        self.h = tuple(float(x) for x in h)
        self.shape = tuple(int(s) for s in shape)
        self.ndim = len(self.shape)
        self.ncfg = self.ndim // 2
        self.fbg = np.asarray(fbg, dtype=np.float64)
        self.recon = recon
        self.field_mode = field_mode
        self.E_prescribed = None if E_prescribed is None else np.asarray(E_prescribed, np.float64)
        self.vbar = [scheme.exact_vbar(self.lower[v], self.h[v], self.shape[v])
                     for v in range(self.ncfg, self.ndim)]
        self.dv_volume = float(np.prod(self.h[self.ncfg:]))

    # -- ComputeInstantaneousConstraints (Alg.5)
    def constraints(self, f):
        """Cell-averaged field on the configuration mesh (no ghosts), shape (ncfg, *cfg)."""
        if self.field_mode == "prescribed":
            return self.E_prescribed.copy()
        rho = field.moment_rho(f, self.dv_volume)
        if self.ncfg == 2:                                   # 2D+2V self-consistent field (N3)
            from . import field2d
            return field2d.efield_from_rho_2d(rho, self.h[0], self.h[1])
        return field.efield_from_rho(rho, self.h[0])[None, :]

    def ghosted_field(self, E):
        return [field.ghost_periodic(E[d]) for d in range(self.ncfg)]

    def rhs(self, f, E, E_bc):
        fg = fill_ghosts_uniform(f, self.ghosted_field(E_bc), self.fbg)
        return scheme.rhs(fg, self.vbar, self.ghosted_field(E), self.h, self.recon)

    def step(self, f_old, E_bc, dt):
        """One RK4 step (Alg.5 with one hierarchy / one level).  ``E_bc`` is the E of the
        previous constraint evaluation, E(f_old) (reading #6b).  Returns (f_new, E(f_new), F_acc):
        the step ends with Alg.5's ComputeInstantaneousConstraints(f_new)."""
        k = np.zeros_like(f_old)
        F_acc = None
        for s in range(4):
            f_pred = f_old + RK_ALPHA[s] * dt * k                      # Alg.2
            E = self.constraints(f_pred)                               # Alg.5
            k, F = self.rhs(f_pred, E, E_bc)                           # Alg.3 (BC uses E_bc)
            F_acc = [RK_B[s] * Fd for Fd in F] if F_acc is None else \
                [Fa + RK_B[s] * Fd for Fa, Fd in zip(F_acc, F)]
            E_bc = E
        f_new = f_old + dt * scheme.divergence(F_acc, self.h)         # Alg.4
        return f_new, self.constraints(f_new), F_acc                   # Alg.5: constraints(f_new)

    def run(self, f0, dt, nsteps, callback=None):
        """Advance nsteps; callback(n, f_n, E(f_n)) after each step (E = stage-1 field)."""
        f = np.array(f0, dtype=np.float64, copy=True)
        E_bc = self.constraints(f)          # first evaluation (ghost-independent here)
        for n in range(nsteps):
            f, E_bc, _ = self.step(f, E_bc, dt)
            if callback is not None:
                callback(n + 1, f, self.constraints(f))
        return f, E_bc


def problem_for(workload, recon=scheme.CENTERED4, ratio=None):
    """Build the UniformProblem of a BASELINE.json workload (inputs only come from ``inputs``)."""
    import inputs
    h = inputs.spacing(workload, ratio)
    shape = tuple(workload.ncells[d] * (ratio[d] if ratio else 1) for d in range(workload.ndim))
    fbg = inputs.background_profile(workload, ratio)
    Ep = inputs.prescribed_field(workload, ratio) if workload.field == "prescribed" else None
    return UniformProblem(workload.lower, h, shape, fbg, recon, workload.field, Ep)
