"""Pins of the 2D+2V (NEXT row N3) oracle pieces: the 2D periodic Poisson solve (oracle/field2d.py,
reading #32) and the 2D+2V hierarchy (oracle/amr4.py): what the paper and the mathematics fix
-- a single-mode closed form, reduction to the pinned 1D solve, exactness of the dimension-by-
dimension linear5 interpolation on tensor quartics, Alg.8 == Alg.6 (the two
reductions are algebraically the same), f == 1 => rho = 1 - velocity volume, Alg.7 sub-patches
tiling exactly, a fine level covering the domain reducing to the uniform fine run, and the
composite mass conserved to round-off when nothing crosses the velocity boundary."""
import itertools

import numpy as np
import pytest

import inputs
from inputs.hierarchies import random_hierarchy_4d
from oracle import amr4, boxes, field, field2d, interp, uniform

G = 2


# --------------------------------------------------------------------------- 2D Poisson
def _lam(theta):
    """Symbol of the 1D operator 30 - 16 (S + S^-1) + (S^2 + S^-2) on e^{i theta i}."""
    return 30.0 - 32.0 * np.cos(theta) + 2.0 * np.cos(2.0 * theta)


@pytest.mark.parametrize("nx,ny,p,q", [(16, 12, 1, 2), (10, 20, 3, 1), (8, 8, 4, 3)])
def test_poisson2d_single_mode_closed_form(nx, ny, p, q):
    dx, dy = 0.37, 0.21
    i, k = np.arange(nx)[:, None], np.arange(ny)[None, :]
    tx, ty = 2 * np.pi * p / nx, 2 * np.pi * q / ny
    rho = 0.7 * np.cos(tx * i) * np.cos(ty * k) + 0.25             # + constant (projected away)
    amp = 12.0 * 0.7 / (_lam(tx) / dx ** 2 + _lam(ty) / dy ** 2)
    phi = field2d.solve_potential_2d(rho, dx, dy)
    np.testing.assert_allclose(phi, amp * np.cos(tx * i) * np.cos(ty * k), rtol=0, atol=1e-12 * amp)
    E = field2d.efield_from_potential_2d(phi, dx, dy)
    ex = amp * (16 * np.sin(tx) - 2 * np.sin(2 * tx)) / (12 * dx) * np.sin(tx * i) * np.cos(ty * k)
    ey = amp * (16 * np.sin(ty) - 2 * np.sin(2 * ty)) / (12 * dy) * np.cos(tx * i) * np.sin(ty * k)
    np.testing.assert_allclose(E[0], ex, rtol=0, atol=1e-11 * max(1.0, np.abs(ex).max()))
    np.testing.assert_allclose(E[1], ey, rtol=0, atol=1e-11 * max(1.0, np.abs(ey).max()))


def test_poisson2d_y_independent_reduces_to_1d():
    rng = np.random.default_rng(3)
    nx, ny, dx, dy = 24, 9, 0.3, 0.45
    r1 = rng.standard_normal(nx)
    E = field2d.efield_from_rho_2d(np.repeat(r1[:, None], ny, axis=1), dx, dy)
    E1 = field.efield_from_rho(r1, dx)
    np.testing.assert_allclose(E[0], np.repeat(E1[:, None], ny, axis=1), rtol=0, atol=1e-12)
    np.testing.assert_allclose(E[1], 0.0, atol=1e-12)
    # Gauss: the cell-averaged field has zero mean on the periodic domain
    E2 = field2d.efield_from_rho_2d(rng.standard_normal((nx, ny)), dx, dy)
    assert abs(E2[0].mean()) < 1e-13 and abs(E2[1].mean()) < 1e-13


# --------------------------------------------------------------------------- interpolation
def test_refine_patch_4d_exact_on_tensor_quartics():
    # linear5 reproduces cell averages of degree-4 polynomials along each dimension; done
    # dimension by dimension it reproduces tensor products of them
    rng = np.random.default_rng(5)
    n, R = (3, 2, 2, 3), (2, 4, 2, 2)
    polys, coarse, fine = [], [], []
    for d in range(4):
        c = rng.standard_normal(5)
        P = np.polynomial.polynomial.Polynomial(c).integ()
        ec = 0.3 * np.arange(-G, n[d] + G + 1)
        ef = 0.3 * np.arange(0, n[d] * R[d] + 1) / R[d]
        coarse.append((P(ec[1:]) - P(ec[:-1])) / np.diff(ec))
        fine.append((P(ef[1:]) - P(ef[:-1])) / np.diff(ef))
    cg = np.einsum("a,b,c,d->abcd", *coarse)
    ref = np.einsum("a,b,c,d->abcd", *fine)
    got = amr4.refine_patch_4d(cg, R, interp.LINEAR5)
    np.testing.assert_allclose(got, ref, rtol=0, atol=1e-11 * np.abs(ref).max())


# --------------------------------------------------------------------------- hierarchies
W4 = inputs.scaled(inputs.get("C5P"), (8, 8, 8, 8), (8, 8, 4, 8))


def _hier(rat, lb, w=W4, fbg_fn=None):
    fbg_fn = fbg_fn or (lambda r: inputs.background_profile(w, r))
    return amr4.Hierarchy4(w.lower, inputs.spacing(w), w.ncells, lb, rat, fbg_fn)


def _random_data(H, seed):
    rng = np.random.default_rng(seed)
    data = H.new_data()
    for l, lvl in enumerate(H.levels):
        for p, b in enumerate(lvl.boxes):
            amr4._interior(data[l][p])[...] = inputs.initial_cell_averages(W4, lvl.ratio, b) * (
                1.0 + 0.1 * rng.standard_normal(boxes.size(b)))
    return data


def _random_E(H, seed):
    rng = np.random.default_rng(seed)
    return [0.2 * rng.standard_normal((2,) + tuple(H.ncells0[d] * lvl.ratio[d] for d in range(2))) for lvl in H.levels]


@pytest.mark.parametrize("seed", range(3))
def test_subpatches_tile_each_patch_4d(seed):
    # Alg.7 in 4D: sub-patches disjoint, inside the patch, not covered by a finer
    # level, and together with the finer footprints they cover the patch cell by cell
    rat, lb = random_hierarchy_4d(seed)
    H = _hier(rat, lb)
    for l, lvl in enumerate(H.levels[:-1]):
        fl = H.levels[l + 1]
        rr = tuple(f // c for f, c in zip(fl.ratio, lvl.ratio))
        for b in lvl.boxes:
            cnt = np.zeros(boxes.size(b), int)
            for s in boxes.compute_sub_patches(b, l, H.levels):
                assert boxes.contains_box(b, s)
                cnt[amr4._sl(s, b[0])] += 1
            cov = np.zeros(boxes.size(b), bool)
            for fb in fl.boxes:
                cb = boxes.intersect(boxes.coarsen(fb, rr), b)
                if not boxes.is_empty(cb):
                    cov[amr4._sl(cb, b[0])] = True
            assert np.all(cnt[~cov] == 1) and np.all(cnt[cov] == 0)


@pytest.mark.parametrize("seed", range(3))
def test_subpatch_reduction_equals_mask_reduction_4d(seed):
    # refining the 2D partial sums (Alg.8) == summing refined 4D data with a mask
    # (Alg.6), since the interpolation is linear and acts on configuration dims only
    rat, lb = random_hierarchy_4d(seed)
    H = _hier(rat, lb)
    data = _random_data(H, seed)
    amr4.fill_ghosts(H, data, _random_E(H, seed))
    a = amr4.subpatch_moment(H, data)
    b = amr4.mask_moment(H, data)
    np.testing.assert_allclose(a, b, rtol=0, atol=1e-13 * np.abs(b).max())


def test_unit_distribution_gives_closed_form_density():
    # f == 1 (and unperturbed profile 1): rho = 1 - (v_x range)(v_y range) on every finest cell
    rat, lb = random_hierarchy_4d(1)
    H = _hier(rat, lb, fbg_fn=lambda r: np.ones((8 * r[2] + 4, 8 * r[3] + 4)))
    data = H.new_data()
    for lvl_d in data:
        for a in lvl_d:
            amr4._interior(a)[...] = 1.0
    amr4.fill_ghosts(H, data, _random_E(H, 2))
    _, rho = amr4.constraints(H, data)
    np.testing.assert_allclose(rho, 1.0 - 12.0 * 12.0, rtol=0, atol=1e-12)


def test_fine_level_covering_domain_equals_uniform_fine_run():
    # a level 1 covering the whole domain: level 1 evolves as the uniform fine problem (the coarse
    # level contributes no sub-patch to the reduction, its ghosts come from siblings / periodic
    # images and the characteristic condition only)
    w = W4
    rat = [(1, 1, 1, 1), (2, 2, 2, 2)]
    lb = [[((0, 0, 0, 0), (7, 7, 7, 7))], [((0, 0, 0, 0), (15, 7, 7, 15)), ((0, 8, 0, 0), (15, 15, 7, 15)),
                                            ((0, 0, 8, 0), (15, 15, 15, 15))]]
    H = _hier(rat, lb)
    data = H.new_data()
    for l, lvl in enumerate(H.levels):
        for p, b in enumerate(lvl.boxes):
            amr4._interior(data[l][p])[...] = inputs.initial_cell_averages(w, lvl.ratio, b)
    E = amr4.start(H, data)
    dt = inputs.fixed_dt(w, (2, 2, 2, 2))
    new, _, _ = amr4.step(H, data, E, dt)
    prob = uniform.problem_for(w, ratio=(2, 2, 2, 2))
    f0 = inputs.initial_cell_averages(w, (2, 2, 2, 2))
    ref, _ = prob.run(f0, dt, 1)
    got = np.empty_like(ref)
    for p, b in enumerate(H.levels[1].boxes):
        got[amr4._sl(b, (0, 0, 0, 0))] = amr4._interior(new[1][p])
    np.testing.assert_allclose(got, ref, rtol=0, atol=1e-13 * np.abs(ref).max())


def _compact_v(w, ratio, b):
    """(1 + 0.05 cos x cos y) g(v_x) g(v_y), g = (1 - (v/0.45)^2)^4 on |v| < 0.45 (exactly 0
    outside): cell averages by 8-point Gauss-Legendre per cell."""
    gx, gw = np.polynomial.legendre.leggauss(8)

    def avg(edges, fn):
        a, c = edges[:-1, None], edges[1:, None]
        pts = 0.5 * (a + c) + 0.5 * (c - a) * gx[None, :]
        return 0.5 * np.sum(gw[None, :] * fn(pts), axis=1)
    e = [inputs.cell_edges(w, d, ratio[d], b[0][d], b[1][d]) for d in range(4)]
    cx = avg(e[0], np.cos)
    cy = avg(e[1], np.cos)
    g = lambda v: np.where(np.abs(v) < 0.45, (1.0 - (v / 0.45) ** 2) ** 4, 0.0)   # noqa: E731
    return (1.0 + 0.05 * cx[:, None, None, None] * cy[None, :, None, None]) * \
        avg(e[2], g)[None, None, :, None] * avg(e[3], g)[None, None, None, :]


def test_two_level_composite_mass_conserved():
    # SURVEY 8(c)-III mass: no flux crosses the velocity boundary (f vanishes on the 4 cells next
    # to it through all stages -- a stage widens the support by 2 cells -- and the incoming profile
    # is 0), so the composite mass -- level 0 after average-down -- is conserved to round-off
    # through the refluxed RK4 step (Alg.4 flux substitution in 4D)
    w = inputs.scaled(inputs.get("C5P"), (8, 8, 24, 24), (8, 8, 24, 24))
    rat = [(1, 1, 1, 1), (2, 2, 2, 2)]
    lb = [[((0, 0, 0, 0), (7, 7, 23, 23))], [((4, 2, 18, 20), (11, 9, 29, 27))]]
    H = amr4.Hierarchy4(w.lower, inputs.spacing(w), w.ncells, lb, rat,
                        lambda r: np.zeros((24 * r[2] + 4, 24 * r[3] + 4)))
    data = H.new_data()
    for l, lvl in enumerate(H.levels):
        for p, b in enumerate(lvl.boxes):
            amr4._interior(data[l][p])[...] = _compact_v(w, lvl.ratio, b)
    amr4.average_down(H, data)
    vol = np.prod(inputs.spacing(w))
    M0 = amr4._interior(data[0][0]).sum() * vol
    E = amr4.start(H, data)
    dt = inputs.fixed_dt(w, (2, 2, 2, 2))
    new, E, _ = amr4.step(H, data, E, dt)
    f0 = amr4._interior(new[0][0])
    assert np.all(f0[:, :, :2, :] == 0.0) and np.all(f0[:, :, -2:, :] == 0.0)
    M = f0.sum() * vol
    assert abs(M - M0) < 1e-13 * M0, (M - M0) / M0
    # the fine patch sits on the support: the step moved mass across the coarse-fine interface
    assert np.max(np.abs(amr4._interior(new[1][0]) - amr4._interior(data[1][0]))) > 1e-6
