"""Pins of the oracle's single-level discretisation (oracle/scheme.py, oracle/uniform.py)
against what the paper and mathematics fix: golden constants, exactness on polynomial data,
free-stream preservation, exact free-streaming solutions (convergence order), the RK4
amplification factor of a Fourier mode, and the 4D operator reducing to the 1D+1V one."""
import json
import os

import numpy as np
import pytest
from scipy import special

import inputs
from oracle import scheme, uniform, field

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_constants.json")))
G = 2


def test_golden_constants():
    assert list(uniform.RK_ALPHA) == GOLD["rk4"]["alpha"]
    np.testing.assert_allclose(uniform.RK_B, GOLD["rk4"]["b"], rtol=0, atol=0)
    f = np.array([3.0, -1.0, 2.0, 7.0])
    L = scheme.third_order_left(f[0], f[1], f[2])
    assert L == pytest.approx(np.dot(GOLD["third_order_left"]["coeffs"], f[:3]) / 6.0, abs=1e-15)
    R = scheme.third_order_right(f[1], f[2], f[3])
    assert R == pytest.approx(np.dot(GOLD["third_order_right"]["coeffs"], f[1:]) / 6.0, abs=1e-15)
    assert scheme.EPS_WENO == GOLD["weno5"]["eps"]


def _poly_cell_avgs(coeffs, edges):
    """Exact cell averages of the polynomial sum c_k x^k."""
    P = np.polynomial.polynomial.Polynomial(coeffs).integ()
    return (P(edges[1:]) - P(edges[:-1])) / np.diff(edges)


@pytest.mark.parametrize("deg", [0, 1, 2, 3])
def test_centered4_face_exact_on_cubics(deg):
    # the 4th-order face average of cell averages of a cubic is the exact point value
    rng = np.random.default_rng(deg)
    c = rng.standard_normal(deg + 1)
    edges = np.array([-2.0, -1.0, 0.0, 1.0, 2.0]) * 0.37
    u = _poly_cell_avgs(c, edges)
    face = scheme.face_average(u[0], u[1], u[2], u[3], scheme.CENTERED4, 1.0)
    assert face == pytest.approx(np.polynomial.polynomial.polyval(0.0, c), abs=1e-14)


def test_face_textbook_values():
    assert scheme.face_average(1.0, 2.0, 3.0, 4.0, scheme.CENTERED4, 1) == pytest.approx(2.5, abs=1e-15)
    assert scheme.face_average(0.0, 0.0, 0.0, 1.0, scheme.CENTERED4, 1) == pytest.approx(-1 / 12, abs=1e-15)


def test_upwind_weights_favour_upwind_stencil():
    # a jump between cells i+1 and i+2: the left (upwind for v>0) stencil is smooth and must
    # dominate, giving ~ the left third-order value 0; for v<0 the right stencil dominates.
    pos = scheme.face_average(0.0, 0.0, 0.0, 1.0, scheme.UPWIND, +1.0)
    neg = scheme.face_average(0.0, 0.0, 0.0, 1.0, scheme.UPWIND, -1.0)
    assert abs(pos) < 1e-12
    assert neg == pytest.approx(-1.0 / 6.0, abs=1e-11)
    # smooth symmetric data -> equal indicators -> ideal weights -> centered value
    for upw in (1.0, -1.0):
        assert scheme.face_average(1.0, 2.0, 3.0, 4.0, scheme.UPWIND, upw) == pytest.approx(2.5, abs=1e-14)
    wl, wr = scheme.provisional_weights(0.3, 0.1, 0.7, 0.2)
    assert wl + wr == pytest.approx(1.0, abs=1e-15)


def _rand_setup(shape, seed):
    rng = np.random.default_rng(seed)
    ndim = len(shape)
    ncfg = ndim // 2
    h = tuple(rng.uniform(0.1, 0.5, ndim))
    vbar = [scheme.exact_vbar(rng.uniform(-3, -1), h[ncfg + d], shape[ncfg + d]) for d in range(ncfg)]
    cfg_g = tuple(s + 2 * G for s in shape[:ncfg])
    E = [rng.standard_normal(cfg_g) for _ in range(ncfg)]
    return h, vbar, E


@pytest.mark.parametrize("shape", [(8, 9), (5, 4, 6, 5)])
@pytest.mark.parametrize("recon", [scheme.CENTERED4, scheme.UPWIND])
def test_free_stream_preservation(shape, recon):
    # constant f => every flux difference cancels exactly => k == 0 bitwise (any E, any v)
    h, vbar, E = _rand_setup(shape, 1)
    fg = np.full(tuple(s + 2 * G for s in shape), 0.731)
    k, F = scheme.rhs(fg, vbar, E, h, recon)
    assert np.all(k == 0.0)


def _free_stream_exact(w, n, t):
    """Exact cell averages of M(v)(1 + a cos(k(x - v t))) (closed form with complex erf)."""
    ex = inputs.cell_edges(w, 0, n[0] // w.ncells[0])
    ev = inputs.cell_edges(w, 1, n[1] // w.ncells[1])
    dx, dv = ex[1] - ex[0], ev[1] - ev[0]
    k, a = w.k[0], w.alpha
    xc = 0.5 * (ex[1:] + ex[:-1])
    Sx = np.sin(k * dx / 2) / (k * dx / 2)
    beta = k * t
    Mbar = inputs.workloads.v_profile_cell_average("landau", ev)
    z = 0.5 * np.exp(-beta ** 2 / 2) * (special.erf((ev[1:] + 1j * beta) / np.sqrt(2))
                                        - special.erf((ev[:-1] + 1j * beta) / np.sqrt(2))) / dv
    return Mbar[None, :] + a * Sx * np.real(np.exp(1j * k * xc)[:, None] * z[None, :])


@pytest.mark.parametrize("recon,order", [(scheme.CENTERED4, 3.85), (scheme.UPWIND, 3.85)])
def test_free_streaming_convergence(recon, order):
    # E == 0: exact solution f0(x - v t, v); 4th-order in space, RK4 in time
    base = inputs.scaled(inputs.get("C1"), (32, 32))
    from dataclasses import replace
    base = replace(base, alpha=0.05)
    errs = []
    T = 0.8
    for n in (32, 64, 128):
        w = inputs.scaled(base, (n, n))
        w = replace(w, ncells=(n, n))
        h = inputs.spacing(w)
        prob = uniform.UniformProblem(w.lower, h, (n, n), inputs.background_profile(w), recon,
                                      "prescribed", np.zeros((1, n)))
        nst = int(round(T / (0.4 * h[0] / 6.0)))
        dt = T / nst
        f, _ = prob.run(inputs.initial_cell_averages(w), dt, nst)
        errs.append(np.max(np.abs(f - _free_stream_exact(w, (n, n), T))))
    rates = np.log2(np.array(errs[:-1]) / np.array(errs[1:]))
    assert np.all(rates > order), (errs, rates)


def test_rk4_amplification_of_a_fourier_mode():
    # f_ij = 1 + eps cos(theta i) g_j, E == 0, background 1 (so the perturbation has zero ghost
    # values).  The mode evolves by the linear system u' = lam_x M u with lam_x the centered-4
    # FV x-symbol -(1 - e^{-i theta}) F(theta)/dx and M = diag(vbar) + (dv/24) C (C the centered
    # difference of the transverse term, truncated at the v-boundary).  One RK4 step is
    # u1 = (I + Z + Z^2/2 + Z^3/6 + Z^4/24) u0 with Z = dt lam_x M  (P:389-398 tableau).
    nx, nv = 16, 6
    h = (0.3, 0.5)
    lower = (0.0, -1.5)
    theta = 2 * np.pi * 3 / nx
    i = np.arange(nx)
    g = np.array([0.3, -0.2, 1.0, 0.5, 0.1, -0.4])
    f0 = 1.0 + 0.1 * np.cos(theta * i)[:, None] * g[None, :]
    prob = uniform.UniformProblem(lower, h, (nx, nv), np.ones(nv + 4), scheme.CENTERED4, "prescribed",
                                  np.zeros((1, nx)))
    dt = 0.05
    f1, _, _ = prob.step(f0, np.zeros((1, nx)), dt)
    Fsym = (-np.exp(-1j * theta) + 7 + 7 * np.exp(1j * theta) - np.exp(2j * theta)) / 12
    lam = -(1 - np.exp(-1j * theta)) * Fsym / h[0]
    vbar = lower[1] + (np.arange(nv) + 0.5) * h[1]
    C = np.diag(np.ones(nv - 1), 1) - np.diag(np.ones(nv - 1), -1)
    M = np.diag(vbar) + (h[1] / 24.0) * C
    Z = dt * lam * M
    P = np.eye(nv) + Z + Z @ Z / 2 + Z @ Z @ Z / 6 + Z @ Z @ Z @ Z / 24
    u1 = P @ g.astype(complex)
    expect = 1.0 + 0.1 * np.real(np.exp(1j * theta * i)[:, None] * u1[None, :])
    np.testing.assert_allclose(f1, expect, rtol=0, atol=5e-15)


def test_rk4_scalar_factor():
    # S:602 [DERIVED]: R(-0.1) = 0.9048375
    z = -0.1
    assert 1 + z + z ** 2 / 2 + z ** 3 / 6 + z ** 4 / 24 == pytest.approx(0.9048375, abs=1e-7)


def test_4d_operator_reduces_to_1d1v():
    # f(x,y,vx,vy) = g(x,vx) h(vy), Ey == 0, Ex = Ex(x): the 4D RHS equals the 1D+1V RHS of g
    # times h (y-fluxes and vy-fluxes cancel), and the same with the roles of (x,vx),(y,vy)
    # swapped -- this exercises every axis of the generic operator against the pinned 1D+1V one.
    rng = np.random.default_rng(3)
    nx, ny, nvx, nvy = 6, 5, 7, 6
    h = (0.3, 0.4, 0.25, 0.35)
    for recon in (scheme.CENTERED4, scheme.UPWIND):
        gg = rng.uniform(0.5, 1.5, (nx + 4, nvx + 4))
        # UPWIND weights are not scale invariant (eps): use a constant factor there
        hh = rng.uniform(0.5, 1.5, nvy + 4) if recon == scheme.CENTERED4 else np.ones(nvy + 4)
        Ex = rng.standard_normal(nx + 4)
        vbx = scheme.exact_vbar(-1.0, h[2], nvx)
        vby = scheme.exact_vbar(-0.7, h[3], nvy)
        f4 = gg[:, None, :, None] * hh[None, None, None, :] * np.ones((1, ny + 4, 1, 1))
        E4 = [np.repeat(Ex[:, None], ny + 4, 1), np.zeros((nx + 4, ny + 4))]
        k4, _ = scheme.rhs(f4, [vbx, vby], E4, h, recon)
        k2, _ = scheme.rhs(gg, [vbx], [Ex], (h[0], h[2]), recon)
        expect = k2[:, None, :, None] * hh[None, None, G:-G, None].reshape(1, 1, 1, nvy)
        np.testing.assert_allclose(k4, np.broadcast_to(expect, k4.shape), rtol=1e-13, atol=1e-13)
        # swapped roles: depends on (y, vy) only
        gy = rng.uniform(0.5, 1.5, (ny + 4, nvy + 4))
        hx = rng.uniform(0.5, 1.5, nvx + 4) if recon == scheme.CENTERED4 else np.ones(nvx + 4)
        Ey = rng.standard_normal(ny + 4)
        f4b = np.ones((nx + 4, 1, 1, 1)) * gy[None, :, None, :] * hx[None, None, :, None]
        E4b = [np.zeros((nx + 4, ny + 4)), np.repeat(Ey[None, :], nx + 4, 0)]
        k4b, _ = scheme.rhs(f4b, [vbx, vby], E4b, h, recon)
        k2b, _ = scheme.rhs(gy, [vby], [Ey], (h[1], h[3]), recon)
        expect = k2b[None, :, None, :] * hx[None, None, G:-G, None]
        np.testing.assert_allclose(k4b, np.broadcast_to(expect, k4b.shape), rtol=1e-13, atol=1e-13)


def test_landau_damping_rate_c1_grid():
    # linear Landau damping k=0.5: omega = 1.415662, gamma = -0.153359 (SURVEY App. A6,
    # Z-function root); run the C1 grid to t = 20, fit the peaks of ||E||_2.
    w = inputs.get("C1")
    prob = uniform.problem_for(w)
    dt = inputs.fixed_dt(w)
    ts, es = [], []
    prob.run(inputs.initial_cell_averages(w), dt, int(20 / dt),
             lambda n, f, E: (ts.append(n * dt), es.append(np.sqrt(np.sum(E ** 2) * prob.h[0]))))
    ts, es = np.array(ts), np.array(es)
    pk = [i for i in range(1, len(es) - 1) if es[i] > es[i - 1] and es[i] > es[i + 1] and ts[i] > 1]
    gamma = np.polyfit(ts[pk], np.log(es[pk]), 1)[0]
    omega = np.pi / np.mean(np.diff(ts[pk]))
    assert abs(gamma - (-0.153359)) <= 0.005
    assert abs(omega - 1.415662) <= 0.01


def test_mass_ledger_uniform():
    # periodic x: the mass changes only by the time-integrated v-boundary flux of F*
    w = inputs.get("C1")
    prob = uniform.problem_for(w)
    f = inputs.initial_cell_averages(w)
    E_bc = prob.constraints(f)
    dt = inputs.fixed_dt(w)
    dx, dv = prob.h
    for _ in range(5):
        m0 = f.sum() * dx * dv
        f, E_bc, F = prob.step(f, E_bc, dt)
        ledger = dt * dx * (np.sum(F[1][:, -1]) - np.sum(F[1][:, 0]))
        assert abs(f.sum() * dx * dv - m0 - ledger) < 1e-14


def test_moment_of_maxwellian_closed_form():
    # rho_i = 1 - (1 + a S_x cos(k x_i)) (Phi(vmax) - Phi(vmin)) exactly for exact cell averages
    w = inputs.get("C1")
    f = inputs.initial_cell_averages(w)
    dv = inputs.spacing(w)[1]
    rho = field.moment_rho(f, dv)
    ex = inputs.cell_edges(w, 0)
    xfac = (np.sin(w.k[0] * ex[1:]) - np.sin(w.k[0] * ex[:-1])) / (w.k[0] * np.diff(ex))
    expect = 1.0 - (1.0 + w.alpha * xfac) * special.erf(6 / np.sqrt(2))
    np.testing.assert_allclose(rho, expect, rtol=0, atol=1e-14)
    # 2D+2V (C5 shape, small grid)
    w5 = inputs.scaled(inputs.get("C5"), (8, 8, 16, 16))
    f5 = inputs.initial_cell_averages(w5)
    h5 = inputs.spacing(w5)
    rho5 = field.moment_rho(f5, h5[2] * h5[3])
    e0, e1 = inputs.cell_edges(w5, 0), inputs.cell_edges(w5, 1)
    cx = (np.sin(e0[1:]) - np.sin(e0[:-1])) / np.diff(e0)
    cy = (np.sin(e1[1:]) - np.sin(e1[:-1])) / np.diff(e1)
    expect5 = 1.0 - (1.0 + 0.01 * cx[:, None] * cy[None, :]) * special.erf(6 / np.sqrt(2)) ** 2
    np.testing.assert_allclose(rho5, expect5, rtol=0, atol=1e-14)


def test_outgoing_extrapolation_exact_on_cubics():
    # reading #6: cubic extrapolation of cell averages (exact for cell averages of cubics)
    rng = np.random.default_rng(7)
    c = rng.standard_normal(4)
    edges = np.arange(-2.0, 5.0) * 0.3
    u = _poly_cell_avgs(c, edges)          # cells -2..3
    g1, g2 = uniform.extrapolate_low(u[2], u[3], u[4], u[5])
    assert g1 == pytest.approx(u[1], abs=1e-13) and g2 == pytest.approx(u[0], abs=1e-13)


def test_velocity_bc_direction_rule():
    # a = -E: low boundary outgoing iff a < 0 (E > 0); high boundary outgoing iff a > 0
    nx, nv = 3, 6
    f = np.arange(nx * nv, dtype=float).reshape(nx, nv) ** 2 * 0.01 + 1.0
    fbg = np.full(nv + 4, -7.0)
    E = np.array([1.0, -1.0, 0.0])
    fg = uniform.fill_ghosts_uniform(f, [np.pad(E, 2, mode="wrap")], fbg)
    g1, _ = uniform.extrapolate_low(f[0, 0], f[0, 1], f[0, 2], f[0, 3])
    assert fg[2, 1] == g1 and fg[2, nv + 2] == -7.0           # E>0: low out, high in
    h1, _ = uniform.extrapolate_low(f[1, -1], f[1, -2], f[1, -3], f[1, -4])
    assert fg[3, 1] == -7.0 and fg[3, nv + 2] == h1           # E<0: low in, high out
    assert fg[4, 1] == -7.0 and fg[4, nv + 2] == -7.0          # E=0: both profile
