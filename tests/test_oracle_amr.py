"""Pins of the oracle's multi-level pieces (oracle/reduction.py, oracle/amr.py):
Alg.6 == Alg.8 on seeded random hierarchies, f = 1 closed form, single-level special case,
CF ghost interpolation exactness, mass ledger across levels, the "fine level covers the
domain" special case, tag formula on linear data."""
import numpy as np
import pytest

import inputs
from inputs.hierarchies import random_hierarchy
from oracle import amr, boxes, field, interp, reduction, scheme, uniform

W = inputs.scaled(inputs.get("C3"), (16, 32), (8, 8))


def _hier(rat, lb, mode=interp.LINEAR5, w=W):
    return amr.Hierarchy(w.lower, inputs.spacing(w), w.ncells, lb, rat,
                         lambda r: inputs.background_profile(w, r), scheme.CENTERED4, mode)


def _fill_ic(H, w=W, noise_seed=None):
    data = H.new_data()
    rng = np.random.default_rng(noise_seed) if noise_seed is not None else None
    for l, lvl in enumerate(H.levels):
        for p, b in enumerate(lvl.boxes):
            v = inputs.initial_cell_averages(w, lvl.ratio, b)
            if rng is not None:
                v = v + 0.01 * rng.standard_normal(v.shape)
            data[l][p][2:-2, 2:-2] = v
    return data


def _zeroE(H):
    return [np.zeros(H.ncells0[0] * lvl.ratio[0]) for lvl in H.levels]


@pytest.mark.parametrize("seed", range(12))
def test_mask_equals_subpatch_reduction(seed):
    rat, lb = random_hierarchy(seed)
    H = _hier(rat, lb)
    data = _fill_ic(H, noise_seed=seed)
    amr.fill_ghosts(H, data, _zeroE(H))
    r1 = reduction.mask_reduce(H.levels, data, H.h0[1], H.ncells0[0])
    r2 = reduction.subpatch_reduce(H.levels, data, H.h0[1], H.ncells0[0])
    np.testing.assert_allclose(r2, r1, rtol=0, atol=1e-12 * np.abs(r1).max())


@pytest.mark.parametrize("seed", range(8))
def test_reduction_of_unity_is_domain_length(seed):
    # f == 1 everywhere (ghosts too): rho = 1 - (vmax - vmin) for any hierarchy (reading #13)
    rat, lb = random_hierarchy(seed)
    H = _hier(rat, lb)
    data = [[np.ones_like(a) for a in lvl] for lvl in H.new_data()]
    for fn in (reduction.mask_reduce, reduction.subpatch_reduce):
        rho = fn(H.levels, data, H.h0[1], H.ncells0[0])
        np.testing.assert_allclose(rho, 1.0 - (W.upper[1] - W.lower[1]), atol=1e-13)


def test_single_level_reduction_is_the_moment():
    lb0 = [boxes.box(*b) for b in inputs.level0_boxes(W)]
    H = _hier([(1, 1)], [lb0])
    data = _fill_ic(H, noise_seed=1)
    amr.fill_ghosts(H, data, _zeroE(H))
    full = np.zeros(W.ncells)
    for p, b in enumerate(H.levels[0].boxes):
        full[b[0][0]:b[1][0] + 1, b[0][1]:b[1][1] + 1] = data[0][p][2:-2, 2:-2]
    rho = reduction.subpatch_reduce(H.levels, data, H.h0[1], H.ncells0[0])
    np.testing.assert_allclose(rho, field.moment_rho(full, H.h0[1]), atol=1e-13)


@pytest.mark.parametrize("mode", [interp.LINEAR5, interp.WENO5])
@pytest.mark.parametrize("seed", [1, 3, 4])
def test_cf_ghosts_exact_for_linear_data(mode, seed):
    # data = cell averages of a + c v (x-periodic) on every level, and the v-boundary profile
    # equal to the same function (E = 0 -> profile ghosts): every fine ghost (SIBLING, COARSE
    # over any number of levels, PHYS) equals the exact cell average, since the conservative
    # interpolation is exact for linear data
    rat, lb = random_hierarchy(seed)
    a, cv = 0.3, -0.02
    w = W

    def vcent(r):
        hv = inputs.spacing(w, r)[1]
        n = w.ncells[1] * r[1]
        return w.lower[1] + (np.arange(-2, n + 2) + 0.5) * hv

    H = amr.Hierarchy(w.lower, inputs.spacing(w), w.ncells, lb, rat,
                      lambda r: a + cv * vcent(r), scheme.CENTERED4, mode)
    data = H.new_data()
    for l, lvl in enumerate(H.levels):
        vc = vcent(lvl.ratio)
        for p, b in enumerate(lvl.boxes):
            data[l][p][2:-2, 2:-2] = (a + cv * vc[b[0][1] + 2: b[1][1] + 3])[None, :]
    amr.fill_ghosts(H, data, _zeroE(H))
    for l, lvl in enumerate(H.levels):
        vc = vcent(lvl.ratio)
        for p, b in enumerate(lvl.boxes):
            exact = np.broadcast_to((a + cv * vc[b[0][1]: b[1][1] + 5])[None, :], data[l][p].shape)
            np.testing.assert_allclose(data[l][p], exact, atol=1e-13)


def _composite_mass(H, data):
    m = 0.0
    for l, lvl in enumerate(H.levels):
        hx, hv = H.h(l)
        for p, b in enumerate(lvl.boxes):
            m += np.sum(reduction.covered_mask(H.levels, l, p) * data[l][p][2:-2, 2:-2]) * hx * hv
    return m


def _ledger(H, F, dt):
    hx, _ = H.h(0)
    nv0 = H.ncells0[1]
    led = 0.0
    for p, b in enumerate(H.levels[0].boxes):
        Fv = F[0][p][1]
        if b[0][1] == 0:
            led -= dt * hx * np.sum(Fv[:, 0])
        if b[1][1] == nv0 - 1:
            led += dt * hx * np.sum(Fv[:, -1])
    return led


@pytest.mark.parametrize("seed", [0, 1, 3, 4])
def test_mass_ledger_two_levels(seed):
    # composite mass changes only by the v-boundary flux (coarse F* substituted by the
    # coarsened fine F* on covered faces, Alg.4) -- conservation to round-off across levels
    rat, lb = random_hierarchy(seed)
    H = _hier(rat, lb)
    data = _fill_ic(H)
    amr.fill_ghosts(H, data, _zeroE(H))
    E_bc, _ = amr.constraints(H, data)
    dt = inputs.fixed_dt(W, H.levels[-1].ratio)
    for _ in range(2):
        m0 = _composite_mass(H, data)
        data, E_bc, F = amr.step(H, data, E_bc, dt)
        assert abs(_composite_mass(H, data) - m0 - _ledger(H, F, dt)) < 2e-14 * abs(m0)


def test_fine_level_covering_domain_equals_uniform_fine_run():
    # level 1 covers the whole domain: its evolution is the single-level fine run (the coarse
    # level is fully covered, contributes nothing to rho and is the average-down of the fine)
    R = (2, 2)
    lb0 = [boxes.box(*b) for b in inputs.level0_boxes(W)]
    fine_boxes = [boxes.box((x, v), (x + 15, v + 31)) for x in (0, 16) for v in (0, 32)]
    H = _hier([(1, 1), R], [lb0, fine_boxes])
    data = _fill_ic(H)
    amr.fill_ghosts(H, data, _zeroE(H))
    E_bc, _ = amr.constraints(H, data)
    wf = inputs.scaled(W, (32, 64))
    prob = uniform.UniformProblem(W.lower, inputs.spacing(wf), (32, 64), inputs.background_profile(wf))
    f = inputs.initial_cell_averages(wf)
    Eu = prob.constraints(f)
    dt = inputs.fixed_dt(W, R)
    for _ in range(3):
        data, E_bc, _ = amr.step(H, data, E_bc, dt)
        f, Eu, _ = prob.step(f, Eu, dt)
    got = np.zeros((32, 64))
    for q, b in enumerate(H.levels[1].boxes):
        got[b[0][0]:b[1][0] + 1, b[0][1]:b[1][1] + 1] = data[1][q][2:-2, 2:-2]
    np.testing.assert_allclose(got, f, rtol=0, atol=1e-13 * np.abs(f).max())
    coarse = np.zeros((16, 32))
    for p, b in enumerate(H.levels[0].boxes):
        coarse[b[0][0]:b[1][0] + 1, b[0][1]:b[1][1] + 1] = data[0][p][2:-2, 2:-2]
    np.testing.assert_allclose(coarse, f.reshape(16, 2, 32, 2).mean(axis=(1, 3)), atol=1e-15)


def test_tags_constant_none_and_linear_threshold():
    hx, hv = 0.2, 0.3
    fg = np.full((12, 14), 0.5)
    assert not amr.tag_cells(fg, hx, hv, 1e-12).any()
    a, b = 0.01, -0.02
    i = np.arange(12)[:, None]
    j = np.arange(14)[None, :]
    fg = 1.0 + a * i + b * j
    d1 = np.sqrt(0.5 * (hx * (2 * a) ** 2 + hv * (2 * b) ** 2))      # delta2 = 0 for linear data
    assert amr.tag_cells(fg, hx, hv, d1 * 0.999).all()
    assert not amr.tag_cells(fg, hx, hv, d1 * 1.001).any()
    spike = np.full((12, 14), 0.5)
    spike[6, 7] = 1.5
    t = amr.tag_cells(spike, hx, hv, 0.05)
    assert t[4, 5] and t[3, 5] and t[4, 4] and t.sum() == 5          # S:579 spike tagged


def test_c3_initial_tags_and_tiles():
    # C3 at t=0 with tol = 0.005 (reading #18): the two-stream maxima of |grad f| are tagged;
    # every tagged cell lies in a tile and tiles hold only dilated tags
    w = inputs.get("C3")
    lb0 = [boxes.box(*b) for b in inputs.level0_boxes(w)]
    H = amr.Hierarchy(w.lower, inputs.spacing(w), w.ncells, [lb0], [(1, 1)],
                      lambda r: inputs.background_profile(w, r))
    data = H.new_data()
    for p, b in enumerate(H.levels[0].boxes):
        data[0][p][2:-2, 2:-2] = inputs.initial_cell_averages(w, (1, 1), b)
    amr.fill_ghosts(H, data, _zeroE(H))
    tags = amr.level0_tags(H, data, w.amr["tol"])
    assert 0 < tags.sum() < tags.size
    assert not amr.level0_tags(H, data, 0.01).any()                  # paper's tol tags nothing
    d = boxes.dilate_tags(tags, w.amr["buffer"], (True, False))
    tiles = boxes.tiles_from_tags(d, w.amr["ratio"], w.amr["tile"])
    cov = np.zeros_like(d)
    for tb in tiles:
        cb = boxes.coarsen(tb, w.amr["ratio"])
        cov[cb[0][0]:cb[1][0] + 1, cb[0][1]:cb[1][1] + 1] = True
        assert d[cb[0][0]:cb[1][0] + 1, cb[0][1]:cb[1][1] + 1].any()
    assert cov[d].all()
