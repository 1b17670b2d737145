"""Pins of oracle/field.py: the periodic Poisson solve and E against the circulant closed form
(single Fourier mode), null-space invariance, and the stencil constants printed in the paper."""
import json
import os

import numpy as np
import pytest

from oracle import field

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_constants.json")))


def test_matrix_matches_printed_stencil():
    A = field.poisson_matrix(8)
    g = GOLD["poisson_stencil"]
    assert A[3, 3] == g["center"] and A[3, 4] == g["pm1"] and A[3, 2] == g["pm1"]
    assert A[3, 5] == g["pm2"] and A[3, 1] == g["pm2"]
    assert np.allclose(A.sum(axis=1), 0.0)             # constants are the null space


@pytest.mark.parametrize("n,m", [(16, 1), (64, 3), (256, 17), (2048, 1)])
def test_single_mode_closed_form(n, m):
    # rho_i = cos(theta i), theta = 2 pi m / n:  phi = 12 dx^2 rho / lambda(theta),
    # lambda = 30 - 32 cos theta + 2 cos 2 theta (circulant eigenvalue);
    # E = -D4 phi = -(16 sin theta - 2 sin 2 theta)/(12 dx) * 12 dx^2/lambda * (-sin(theta i))
    dx = 0.173
    th = 2 * np.pi * m / n
    i = np.arange(n)
    rho = np.cos(th * i) + 0.25                        # + constant: projected out
    lam = 30 - 32 * np.cos(th) + 2 * np.cos(2 * th)
    phi_expect = 12 * dx * dx * np.cos(th * i) / lam
    # the system's condition number is 64 / lambda(2 pi / n): the tolerance scales with it
    cond = 64.0 / (30 - 32 * np.cos(2 * np.pi / n) + 2 * np.cos(4 * np.pi / n))
    tol = 50 * np.finfo(float).eps * cond
    phi = field.solve_potential(rho, dx)
    np.testing.assert_allclose(phi, phi_expect, rtol=0, atol=tol * np.abs(phi_expect).max())
    E = field.efield_from_potential(phi, dx)
    E_expect = (16 * np.sin(th) - 2 * np.sin(2 * th)) / (12 * dx) * (12 * dx * dx / lam) * np.sin(th * i)
    np.testing.assert_allclose(E, E_expect, rtol=0, atol=tol * np.abs(E_expect).max())


def test_null_space_and_mean_zero():
    rng = np.random.default_rng(0)
    rho = rng.standard_normal(40)
    p1 = field.solve_potential(rho, 0.3)
    p2 = field.solve_potential(rho + 7.5, 0.3)
    np.testing.assert_allclose(p1, p2, atol=1e-13)
    assert abs(p1.mean()) < 1e-14
    # the solution satisfies the printed equation with the projected rhs (reading #2: dx^2)
    A = field.poisson_matrix(40)
    np.testing.assert_allclose(A @ p1, 12 * 0.3 ** 2 * (rho - rho.mean()), atol=1e-12)
    E = field.efield_from_potential(p1, 0.3)
    assert abs(E.sum()) < 1e-13                         # Gauss: periodic sum of E vanishes


def test_efield_sign_is_minus_gradient():
    # reading #1: E = -d_x phi; phi = cell averages of sin(x) -> E ~ -cos(x)
    n = 64
    dx = 2 * np.pi / n
    e = dx * np.arange(n + 1)
    phi = (np.cos(e[:-1]) - np.cos(e[1:])) / dx          # cell averages of sin
    E = field.efield_from_potential(phi, dx)
    Eexact = -(np.sin(e[1:]) - np.sin(e[:-1])) / dx       # cell averages of -cos
    np.testing.assert_allclose(E, Eexact, atol=dx ** 4 / 25)   # leading error dx^4/30 |f^(5)|


def test_poisson_rejects_small_n():
    with pytest.raises(ValueError):
        field.poisson_matrix(4)
