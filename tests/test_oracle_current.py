"""Pins of the oracle's current moment (oracle/field.current_density, reading #31): exact for
velocity profiles quadratic in v (the product rule's error starts with the cubic term), the
closed forms of constant and symmetric profiles and of a shifted Maxwellian (j = q n u)."""
import math

import numpy as np
import pytest
from scipy import special

from oracle import field


def _ghosted(cells_x, fbar_v):
    return np.repeat(fbar_v[None, :], cells_x + 4, axis=0)


def _quad_cell_averages(a, b, c, edges):
    """exact cell averages of a + b v + c v^2 on the given edges"""
    lo, hi = edges[:-1], edges[1:]
    F = lambda v: a * v + b * v ** 2 / 2 + c * v ** 3 / 3   # noqa: E731
    return (F(hi) - F(lo)) / (hi - lo)


@pytest.mark.parametrize("nv", [8, 37, 128])
def test_exact_on_quadratic_profiles(nv):
    vlo, vhi = -3.0, 5.0
    dv = (vhi - vlo) / nv
    edges = vlo + dv * np.arange(-2, nv + 3)               # ghosted cells -2 .. nv+1
    a, b, c = 0.7, -0.3, 0.25
    f = _ghosted(3, _quad_cell_averages(a, b, c, edges))
    j = field.current_density(f, vlo, dv, q=-2.0)
    G = lambda v: a * v ** 2 / 2 + b * v ** 3 / 3 + c * v ** 4 / 4   # noqa: E731   int v f dv
    want = -2.0 * (G(vhi) - G(vlo))
    np.testing.assert_allclose(j, want, rtol=0, atol=1e-13 * abs(want) * nv)


def test_constant_and_symmetric_profiles():
    f = _ghosted(4, np.full(20, 1.5))
    j = field.current_density(f, -6.0, 12.0 / 16, q=1.0)
    np.testing.assert_allclose(j, 1.5 * (36.0 - 36.0) / 2, atol=1e-13)
    j2 = field.current_density(f, -2.0, 10.0 / 16, q=1.0)      # v in [-2, 8]
    np.testing.assert_allclose(j2, 1.5 * (64.0 - 4.0) / 2, rtol=1e-14)
    edges = -6.0 + 0.75 * np.arange(-2, 19)
    m = (special.erf(edges[1:] / math.sqrt(2)) - special.erf(edges[:-1] / math.sqrt(2))) / 2 / 0.75
    assert np.max(np.abs(field.current_density(_ghosted(2, m), -6.0, 0.75))) < 1e-15


def test_shifted_maxwellian_closed_form():
    """j = q n u for n M(v - u) (the velocity sum of smooth, decaying cell averages is
    spectrally accurate, so the closed form holds to rounding on every grid)."""
    u, n = 0.8, 1.3
    for nv in (32, 64, 128):
        dv = 20.0 / nv
        edges = -10.0 + dv * np.arange(-2, nv + 3)
        m = (special.erf((edges[1:] - u) / math.sqrt(2)) - special.erf((edges[:-1] - u) / math.sqrt(2))) / 2 / dv
        j = field.current_density(_ghosted(1, n * m), -10.0, dv, q=-1.0)
        assert abs(j[0] - (-n * u)) < 1e-13


def test_hierarchy_first_moment_single_level_equals_uniform():
    """Alg.8 first moment (reading #31) on a level split into patches along v and x: the product
    rule's boundary terms telescope across patch faces, so it equals current_density of the whole
    ghosted level (up to rounding)."""
    import inputs
    from oracle import amr, boxes, interp, reduction, scheme
    w = inputs.scaled(inputs.get("C3"), (16, 32), (8, 8))
    lb = [[boxes.box(*b) for b in inputs.level0_boxes(w)]]
    H = amr.Hierarchy(w.lower, inputs.spacing(w), w.ncells, lb, [(1, 1)],
                      lambda r: inputs.background_profile(w, r), scheme.CENTERED4, interp.LINEAR5)
    f = inputs.initial_cell_averages(w) * (1.0 + 0.1 * inputs.random_field(w.ncells, 3))
    data = H.new_data()
    for p, b in enumerate(H.levels[0].boxes):
        data[0][p][2:-2, 2:-2] = f[b[0][0]:b[1][0] + 1, b[0][1]:b[1][1] + 1]
    amr.fill_ghosts(H, data, [np.full(w.ncells[0], 0.05)])
    got = reduction.subpatch_moment(H.levels, data, H.h0[1], w.ncells[0], first=True, vlo=w.lower[1])
    # the whole level, ghosted, assembled from the patches' filled frames
    fg = np.zeros((w.ncells[0] + 4, w.ncells[1] + 4))
    for p, b in enumerate(H.levels[0].boxes):
        fg[b[0][0]:b[1][0] + 5, b[0][1]:b[1][1] + 5] = data[0][p]
    want = -field.current_density(fg, w.lower[1], H.h0[1], q=-1.0)
    np.testing.assert_allclose(got, want, rtol=0, atol=1e-13 * np.abs(want).max())
