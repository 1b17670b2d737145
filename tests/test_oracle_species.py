"""Pins of the multi-species oracle (oracle/species.py): one electron species reduces to
the single-hierarchy advance; splitting the electrons into two species of the same q/m is an
exact superposition (the scheme is linear in f for a given field, CENTERED4); the charge density
of ions and electrons with equal densities is the neutral rho_bg."""
import numpy as np

import inputs
from inputs.hierarchies import random_hierarchy
from oracle import amr, boxes, interp, scheme, species

W = inputs.scaled(inputs.get("C3"), (16, 32), (8, 8))


def _hier(rat, lb, scale=1.0):
    return amr.Hierarchy(W.lower, inputs.spacing(W), W.ncells, [[boxes.box(*b) for b in bl] for bl in lb], rat,
                         lambda r: scale * inputs.background_profile(W, r), scheme.CENTERED4, interp.LINEAR5)


def _data(H, scale=1.0):
    d = H.new_data()
    for l, lvl in enumerate(H.levels):
        for p, b in enumerate(lvl.boxes):
            d[l][p][2:-2, 2:-2] = scale * inputs.initial_cell_averages(W, lvl.ratio, b)
    return d


def test_single_electron_species_is_the_hierarchy_advance():
    rat, lb = random_hierarchy(2)
    H1 = _hier(rat, lb)
    d1 = _data(H1)
    amr.fill_ghosts(H1, d1, [np.zeros(W.ncells[0] * r[0]) for r in rat])
    E1, _ = amr.constraints(H1, d1)
    Hs = _hier(rat, lb)
    ds = _data(Hs)
    sp = [species.Species(Hs, -1.0, 1.0)]
    A = species.start(sp, [ds], 1.0)
    dt = inputs.fixed_dt(W, rat[-1])
    for _ in range(2):
        d1, E1, _ = amr.step(H1, d1, E1, dt)
        (ds,), A = species.step(sp, [ds], A, dt, 1.0)
    for l in range(len(rat)):
        for a, b in zip(d1[l], ds[l]):
            np.testing.assert_allclose(b[2:-2, 2:-2], a[2:-2, 2:-2], rtol=0, atol=1e-14)


def test_split_electrons_superpose_exactly():
    rat, lb = random_hierarchy(4)
    H1 = _hier(rat, lb)
    d1 = _data(H1)
    amr.fill_ghosts(H1, d1, [np.zeros(W.ncells[0] * r[0]) for r in rat])
    E1, _ = amr.constraints(H1, d1)
    Ha, Hb = _hier(rat, lb, 0.3), _hier(rat, lb, 0.7)
    da, db = _data(Ha, 0.3), _data(Hb, 0.7)
    sp = [species.Species(Ha, -1.0, 1.0), species.Species(Hb, -1.0, 1.0)]
    A = species.start(sp, [da, db], 1.0)
    dt = inputs.fixed_dt(W, rat[-1])
    for _ in range(2):
        d1, E1, _ = amr.step(H1, d1, E1, dt)
        (da, db), A = species.step(sp, [da, db], A, dt, 1.0)
    for l in range(len(rat)):
        for a, b, c in zip(d1[l], da[l], db[l]):
            np.testing.assert_allclose(b[2:-2, 2:-2] + c[2:-2, 2:-2], a[2:-2, 2:-2], rtol=0, atol=1e-14)


def test_neutral_plasma_charge_density():
    rat, lb = random_hierarchy(1)
    He, Hi = _hier(rat, lb), _hier(rat, lb)
    de, di = _data(He), _data(Hi)
    for H, d in ((He, de), (Hi, di)):
        amr.fill_ghosts(H, d, [np.zeros(W.ncells[0] * r[0]) for r in rat])
    rho = species.charge_density([species.Species(He, -1.0, 1.0), species.Species(Hi, 1.0, 25.0)], [de, di], 0.0)
    np.testing.assert_allclose(rho, 0.0, atol=1e-15)
