"""Pins of oracle/interp.py (linear5, WENO5) against polynomial exactness (exact sub-cell
averages by symbolic integration), conservation, the identity case R=1, the printed constants,
and the SPEC worked example."""
import json
import os
from fractions import Fraction

import numpy as np
import pytest

from oracle import interp

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_constants.json")))


def _exact_avgs(coeffs, a, b):
    P = np.polynomial.polynomial.Polynomial(coeffs).integ()
    return (P(b) - P(a)) / (b - a)


@pytest.mark.parametrize("R", [1, 2, 3, 4])
@pytest.mark.parametrize("deg", [0, 1, 2, 3, 4])
def test_linear5_exact_for_quartics(R, deg):
    rng = np.random.default_rng(10 * R + deg)
    c = rng.standard_normal(deg + 1)
    # coarse cells i-2..i+2 = [m, m+1], m = -2..2 (h = 1); fine cells of cell 0
    u5 = np.array([_exact_avgs(c, m, m + 1.0) for m in range(-2, 3)])
    fine = interp.linear5_1d(u5, R)
    expect = np.array([_exact_avgs(c, s / R, (s + 1.0) / R) for s in range(R)])
    np.testing.assert_allclose(fine, expect, atol=1e-12)


def test_linear5_quintic_not_exact():
    # order is exactly 5: a pure x^5 is not reproduced (guards against a trivial pass)
    u5 = np.array([_exact_avgs([0, 0, 0, 0, 0, 1], m, m + 1.0) for m in range(-2, 3)])
    fine = interp.linear5_1d(u5, 2)
    expect = np.array([_exact_avgs([0, 0, 0, 0, 0, 1], s / 2, (s + 1.0) / 2) for s in range(2)])
    assert np.max(np.abs(fine - expect)) > 1e-3


@pytest.mark.parametrize("R", [1, 2, 4, 8])
def test_linear5_weight_invariants(R):
    W = interp.linear5_weights_exact(R)
    for row in W:
        assert sum(row) == 1                                     # constants reproduced
    for j in range(5):                                          # conservation per coarse cell
        assert sum(W[s][j] for s in range(R)) / R == (1 if j == 2 else 0)
    if R == 1:
        assert W[0] == (0, 0, 1, 0, 0)


def test_weno5_constants_match_paper():
    assert list(interp.D_IDEAL) == GOLD["weno5"]["d"]
    assert interp.EPS_WENO == GOLD["weno5"]["eps"]


@pytest.mark.parametrize("R", [2, 3, 4])
def test_weno5_constant_and_linear_exact(R):
    np.testing.assert_allclose(interp.weno5_1d(np.full(5, 0.7), R), np.full(R, 0.7), atol=1e-15)
    u5 = np.array([_exact_avgs([0.3, 1.7], m, m + 1.0) for m in range(-2, 3)])
    expect = np.array([_exact_avgs([0.3, 1.7], s / R, (s + 1.0) / R) for s in range(R)])
    np.testing.assert_allclose(interp.weno5_1d(u5, R), expect, atol=1e-13)


def test_weno5_each_candidate_is_quadratic_exact():
    # for quadratic data every candidate stencil is exact, so the combination is exact for any
    # weights -> this pins A^(r), B^(r) (incl. reading #8 B^(0) = 2D_i - D_{i+1}), C^(r) and the
    # sub-cell formula
    for R in (2, 4):
        c = [0.2, -0.5, 0.9]
        u5 = np.array([_exact_avgs(c, m, m + 1.0) for m in range(-2, 3)])
        expect = np.array([_exact_avgs(c, s / R, (s + 1.0) / R) for s in range(R)])
        np.testing.assert_allclose(interp.weno5_1d(u5, R), expect, atol=1e-13)


def test_weno5_spec_example_and_conservation():
    # S:247-249 [DERIVED]: (-2,-1,0,1,2), R=2 -> (-1/4, 1/4)
    np.testing.assert_allclose(interp.weno5_1d(np.array([-2., -1, 0, 1, 2]), 2), [-0.25, 0.25], atol=1e-15)
    rng = np.random.default_rng(5)
    u = rng.standard_normal((100, 5))
    out = interp.weno5_1d(u, 4)
    np.testing.assert_allclose(out.mean(axis=1), u[:, 2], atol=2e-15)


def test_weno5_step_is_nonoscillatory():
    # step data: the smooth candidate dominates, outputs stay within [0,1] to ~1e-12
    out = interp.weno5_1d(np.array([0., 0, 0, 1, 1]), 4)
    assert out.min() > -1e-11 and out.max() < 1e-11
    out = interp.weno5_1d(np.array([0., 0, 1, 1, 1]), 4)
    np.testing.assert_allclose(out, 1.0, atol=1e-11)


@pytest.mark.parametrize("mode", [interp.LINEAR5, interp.WENO5])
def test_2d_bilinear_exact_and_dimension_order(mode):
    # bilinear f = (a + b x)(c + d v): dimension-by-dimension refinement is exact
    Rx, Rv = 4, 2
    ax = np.array([_exact_avgs([0.5, 0.3], m, m + 1.0) for m in range(-2, 3)])
    av = np.array([_exact_avgs([1.2, -0.4], m, m + 1.0) for m in range(-2, 3)])
    block = ax[:, None] * av[None, :]
    for sx in range(Rx):
        for sv in range(Rv):
            val = interp.interp_fine_cell_2d(block, Rx, Rv, sx, sv, mode)
            ex = _exact_avgs([0.5, 0.3], sx / Rx, (sx + 1.0) / Rx) * _exact_avgs([1.2, -0.4], sv / Rv, (sv + 1.0) / Rv)
            assert val == pytest.approx(ex, abs=1e-13)
    # the patch refinement uses the same x-then-v order as the single-cell routine
    rng = np.random.default_rng(2)
    cg = rng.uniform(0.5, 1.5, (7, 8))
    fine = interp.refine_patch_2d(cg, Rx, Rv, mode)
    for i in range(3):
        for j in range(4):
            blk = cg[i: i + 5, j: j + 5]
            for sx in range(Rx):
                for sv in range(Rv):
                    assert fine[i * Rx + sx, j * Rv + sv] == pytest.approx(
                        interp.interp_fine_cell_2d(blk, Rx, Rv, sx, sv, mode), rel=1e-15, abs=1e-15)
